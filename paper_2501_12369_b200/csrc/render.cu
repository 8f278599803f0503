// render.cu — per-tile front-to-back compositing (forward) and its reverse
// traversal (backward) for the DARBF families, hand-written for sm_100a.
//
// Reference semantics: darbs::forward  src/rasterizer.cpp:55-112 (inner loop :85-107)
//                      darbs::backward src/rasterizer.cpp:147-234 (inner loop :175-214)
//
// Design: one CTA of 8 warps per 16x16 tile (the reference's
// kTileSize, so bins are comparable entry for entry); each warp owns an 8x4
// pixel block and walks the tile's depth-sorted list on its own, 32 entries at
// a time.  A lane first tests ONE entry against the warp's pixel block (exact
// minimum of the conic's quadratic form over the block against the splat's
// decision threshold); survivors are compacted through a per-warp shared-memory
// stage and only those are evaluated per pixel.  No CTA-wide barrier, no
// cross-warp dependency, so a warp whose 32 pixels have saturated leaves
// immediately.  Entries culled at block level are still COUNTED (processed[] is
// positional), so per-pixel aux is identical to the reference's.
//
// Threshold decisions (alpha >= 1/255, dm2 vs cutoff, dm2 < 0) are taken in
// FP32 against a per-splat precomputed boundary; when the FP32 value lies
// inside a guard band of that boundary the decision is re-taken in FP64 with
// the reference's own expression order, so integer outputs match the FP64
// reference.
#include <cooperative_groups.h>

#include "family.cuh"

namespace darbs_b200 {

namespace {

constexpr int kWarpsPerCta = 8;
constexpr int kThreads = 32 * kWarpsPerCta;
constexpr unsigned kFull = 0xffffffffu;

// counters (u64 each): 3 = surviving (warp, entry) pairs, 4 = FP64 re-decisions,
// 5 = pixels whose transmittance came within the guard band of the floor.
enum { CNT_SURVIVORS = 3, CNT_EXACT = 4, CNT_TFLOOR = 5 };

// ------------------------------------------------------------------ packing
__global__ void pack_kernel(KParams kp, int64_t n, const float* __restrict__ mu2,
                            const float* __restrict__ conic, const float* __restrict__ opacity,
                            const float* __restrict__ rgb, float4* __restrict__ recs) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    float mx = mu2[2 * i], my = mu2[2 * i + 1];
    float a = conic[3 * i], b = conic[3 * i + 1], c = conic[3 * i + 2];
    float o = opacity[i];
    double ad = a, bd = b, cd = c;
    double thr = family_threshold(kp, (double)o);
    // An indefinite or non-finite conic cannot be culled by the convex block
    // test and may produce dm2 < 0 (rasterizer.cpp:91): force the FP64 path.
    bool pd = (ad > 0.0) && (cd > 0.0) && (ad * cd - bd * bd > 0.0);
    float thr_m = pd ? (float)(thr * (double)kp.scale) : __int_as_float(0x7fc00000);
    float4* r = recs + kRecVecs * i;
    r[0] = make_float4(mx, my, kp.scale * a, kp.scale * (2.0f * b));
    // cull helpers: minimiser slope along the other axis, -B/(2C) and -B/(2A)
    r[1] = make_float4(kp.scale * c, o, thr_m, -b / c);
    r[2] = make_float4(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2], -b / a);
    r[3] = make_float4(a, b, c, 0.f);
}

__global__ void gather_kernel(int64_t k, const int* __restrict__ point_list,
                              const float4* __restrict__ recs, float4* __restrict__ stream) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= k) return;
    const float4* r = recs + kRecVecs * (int64_t)__ldg(point_list + i);
    const float4 v0 = __ldg(r), v1 = __ldg(r + 1), v2 = __ldg(r + 2);
    stream[i] = v0;
    stream[k + i] = v1;
    stream[2 * k + i] = v2;
}

// ------------------------------------------------------------ shared pieces

// Lower bound of m(d) = A dx^2 + B dx dy + C dy^2 over the rectangle of pixel
// centres [X0,X1]x[Y0,Y1] (d measured from the splat centre), for A, C > 0 and
// 4AC > B^2 (the pack kernel sends every other conic down the NaN path).  The
// minimum of a convex quadratic over a box that does not contain the
// unconstrained minimiser lies on an edge facing it; evaluated branch-free:
// candidate 1 = best point of the vertical line through the x-clamped centre,
// candidate 2 = same for the horizontal line; when the centre is inside the
// box both are 0, when it is outside along one axis only the candidate of the
// other axis lies on the facing edge too and is not smaller.
// kx = -B/(2C), ky = -B/(2A) come precomputed with the record.
__device__ __forceinline__ bool block_survives(float mx, float my, float A, float B, float C,
                                               float kx, float ky, float thr, float band2,
                                               float X0, float X1, float Y0, float Y1) {
    const float ex0 = X0 - mx, ex1 = X1 - mx, ey0 = Y0 - my, ey1 = Y1 - my;
    const float dxc = fminf(fmaxf(0.f, ex0), ex1);
    const float dyc = fminf(fmaxf(0.f, ey0), ey1);
    const float dy1 = fminf(fmaxf(kx * dxc, ey0), ey1);
    const float m1 = fmaf(fmaf(A, dxc, B * dy1), dxc, (C * dy1) * dy1);
    const float dx2 = fminf(fmaxf(ky * dyc, ex0), ex1);
    const float m2 = fmaf(fmaf(A, dx2, B * dyc), dx2, (C * dyc) * dyc);
    const float mmin = fminf(m1, m2);
    // Per-pixel decisions can only be positive for m <= thr + band; keep a
    // relative margin for the FP32 rounding of mmin itself.  A NaN threshold
    // (decided in FP64) compares false and survives.
    return !(mmin * 0.9999f > thr + band2);
}

// FP32 generic evaluation of eval() for FAM_GENERIC (kernel.cpp:127-164).
__device__ __forceinline__ void generic_eval(const KParams& kp, float dm2, float& w, float& dw) {
    if (kp.family == DARBS_INVERSE_MULTIQUADRATIC) {
        float base = dm2 / kp.xi + 1.0f;
        float r = rsqrtf(base);
        w = r;
        dw = -0.5f * r / (base * kp.xi);
        return;
    }
    if (dm2 < 1e-30f) {  // kernel.cpp:146-151: every family has f(0) = 1
        w = 1.0f;
        dw = (float)center_dweight_exact(kp);
        return;
    }
    bool b2 = kp.beta == 2.0f;
    float u = b2 ? dm2 / kp.xi : powf(dm2, 0.5f * kp.beta) / kp.xi;
    float du = b2 ? 1.0f / kp.xi : 0.5f * kp.beta * powf(dm2, 0.5f * kp.beta - 1.0f) / kp.xi;
    float f, df;
    switch (kp.family) {
        case DARBS_GAUSSIAN:
            f = expf(-u);
            df = -f;
            break;
        case DARBS_HALF_COSINE:
            f = cosf(u);
            df = -sinf(u);
            break;
        case DARBS_RAISED_COSINE:
            f = 0.5f + 0.5f * cosf(u);
            df = -0.5f * sinf(u);
            break;
        default: {  // DARBS_MODULUS_SINC
            if (u < 1e-4f) {
                f = 1.0f - u * u / 6.0f;
                df = -u / 3.0f;
            } else {
                float s = sinf(u);
                float sgn = (float)((s > 0.f) - (s < 0.f));
                f = fabsf(s) / u;
                df = sgn * (u * cosf(u) - s) / (u * u);
            }
            break;
        }
    }
    w = fminf(fmaxf(f, 0.f), 1.f);
    dw = df * du;
}

// The reference's per-visit logic (rasterizer.cpp:90-95 / :181-187) in FP64 on
// the values the reference would see (the float32 inputs widened), with its
// expression order (conic_dm2 rasterizer.cpp:19-21).  Returns
// { clamped alpha, weight, d weight / d m, flags } with flags bit 0 = the visit
// contributes, bit 1 = alpha_raw < 0.99 (the clamp lets the gradient through,
// rasterizer.cpp:202).  Out of line: taken for a few visits per million.
__device__ __noinline__ float4 exact_decide(const KParams& kp, const float4* __restrict__ recs,
                                            int idx, float fx, float fy) {
    const float4 v0 = __ldg(recs + kRecVecs * (int64_t)idx);
    const float4 v1 = __ldg(recs + kRecVecs * (int64_t)idx + 1);
    const float4 v3 = __ldg(recs + kRecVecs * (int64_t)idx + 3);
    double dx = (double)fx - (double)v0.x, dy = (double)fy - (double)v0.y;
    double a = v3.x, b = v3.y, c = v3.z, o = v1.y;
    double dm2 = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(a, dx), dx),
                                     __dmul_rn(__dmul_rn(__dmul_rn(2.0, b), dx), dy)),
                           __dmul_rn(__dmul_rn(c, dy), dy));
    float4 out = make_float4(0.f, 0.f, 0.f, __int_as_float(0));
    if (!(dm2 >= 0.0)) return out;  // dm2 < 0 (or NaN, which the reference rejects)
    double w, dw;
    eval_exact(kp, dm2, w, dw);
    double alpha_raw = o * w;
    double alpha = fmin(kAlphaClampD, alpha_raw);
    if (alpha < kAlphaSkipD) return out;
    out.x = (float)alpha;
    out.y = (float)w;
    out.z = (float)(dw / (double)kp.scale);
    out.w = __int_as_float(1 | (alpha_raw < kAlphaClampD ? 2 : 0));
    return out;
}

// FP32 decision of one (pixel, entry) visit.  m = scaled squared Mahalanobis
// distance, computed by the caller with a fixed FMA order shared by forward
// and backward so that both passes take identical decisions.  `near` flags a
// value inside the guard band of a threshold (re-decided in FP64 when
// kp.exact); a_raw = opacity * weight, unclamped.
template <int FAM, bool GRAD>
__device__ __forceinline__ void fast_decide(const KParams& kp, float m, float thr, float o,
                                            bool& hit, bool& near, float& a_raw, float& w,
                                            float& dwdm) {
    if constexpr (FAM == FAM_GENERIC) {
        // m == dm2 here (scale 1); thr == cutoff.
        near = !(fabsf(m) > kp.band) || !(fabsf(m - kp.cutoff) > kp.band);
        const bool in_support = !(m < 0.f) && !(m > kp.cutoff);
        generic_eval(kp, fmaxf(m, 0.f), w, dwdm);
        a_raw = o * w;
        near = near || !(fabsf(a_raw - kAlphaSkipF) > 2e-6f);
        if (GRAD) near = near || !(fabsf(a_raw - kAlphaClampF) > 2e-6f);
        hit = in_support && !(fminf(kAlphaClampF, a_raw) < kAlphaSkipF);
    } else {
        const float d = thr - m;
        near = !(fabsf(d) > kp.band);  // also true for a NaN threshold
        hit = d > 0.f;
        if (GRAD) {
            fam_eval<FAM>(m, w, dwdm);
        } else {
            w = fam_weight<FAM>(m);
            dwdm = 0.f;
        }
        a_raw = o * w;
        if (GRAD) near = near || !(fabsf(a_raw - kAlphaClampF) > 2e-6f);
    }
}

__device__ __forceinline__ float quad_m(float A, float B, float C, float dx, float dy) {
    return fmaf(fmaf(A, dx, B * dy), dx, (C * dy) * dy);
}

// One list entry as a lane holds it while testing it against the warp's block.
struct Entry {
    float4 v0, v1, v2;
};

// ---- tile-ordered record streams
// After the sort, gather_kernel copies the three hot vectors of every list
// entry's record into three arrays in LIST order (v0 | v1 | v2, each K float4),
// so that the 8 warps of a tile read their entries with fully coalesced loads
// (4 L1 wavefronts per load instead of one per lane for a gather through the
// point list) and without a dependent index load.
__device__ __forceinline__ void load_entry(Entry& e, int& idx, const float4* __restrict__ stream,
                                           size_t stride, const int* __restrict__ point_list, int k,
                                           int end) {
    if (k < end) {
        e.v0 = __ldg(stream + k);
        e.v1 = __ldg(stream + stride + k);
        e.v2 = __ldg(stream + 2 * stride + k);
        idx = __ldg(point_list + k);
    }
}

// Per-warp survivor queue in shared memory: a ring of CAP entries of three
// float4 { mu.x, mu.y, A, B } { C, opacity, thr_m, list position } { r, g, b,
// splat index }.  Entries that pass the block test are appended in list order;
// the compositing loops consume them in fixed-size groups that never wrap (CAP
// is a multiple of the group size): one chunk is appended between two drains,
// on top of less than one group left over.
template <int CAP>
__device__ __forceinline__ void queue_push(float4* q, int slot, const Entry& e, int pos, int idx) {
    if (slot >= CAP) slot -= CAP;
    q[slot * 3 + 0] = e.v0;
    q[slot * 3 + 1] = make_float4(e.v1.x, e.v1.y, e.v1.z, __int_as_float(pos));
    q[slot * 3 + 2] = make_float4(e.v2.x, e.v2.y, e.v2.z, __int_as_float(idx));
}

// Pads the queue up to a multiple of GROUP with entries no pixel can take (zero
// opacity, threshold -inf, position past every list, splat index -1), so that the
// last, partial group runs through the same unrolled code as the others.
template <int CAP, int GROUP>
__device__ __forceinline__ int queue_pad(float4* q, int head, int qn, int lane) {
    const int pad = (GROUP - qn % GROUP) % GROUP;
    if (lane < pad) {
        int slot = head + qn + lane;
        if (slot >= CAP) slot -= CAP;
        q[slot * 3 + 0] = make_float4(0.f, 0.f, 0.f, 0.f);
        q[slot * 3 + 1] = make_float4(0.f, 0.f, -3.0e38f, __int_as_float(0x7fffffff));
        q[slot * 3 + 2] = make_float4(0.f, 0.f, 0.f, __int_as_float(-1));
    }
    return qn + pad;
}

// Where the survivor list of block `blk` (0..7, the forward's warp index) of a tile
// whose point list is [beg, end) starts: every block owns a region as long as the
// tile's list, the worst case.  8 * K entries of address space; only survivors are
// ever written or read.
__device__ __forceinline__ size_t survivor_list_offset(int beg, int end, int blk) {
    return (size_t)beg * kWarpsPerCta + (size_t)blk * (size_t)(end - beg);
}

// ------------------------------------------------------------------ forward
constexpr int kGroup = 8;  // survivors composited speculatively between two guard-band checks
constexpr int kFwdQueueCap = 40;  // 32 appended per chunk on top of at most kGroup - 1 left over


// A pixel is live while its transmittance is at or above the floor
// (rasterizer.cpp:100 leaves the loop the first time T < 1e-4); lanes outside
// the image start at T = 0 and never take a splat.
struct FwdPixel {
    float T, cr, cg, cb;
    float contrib;  // contributor count, kept in FP32 (exact below 2^24) so a hit costs one FADD
    int proc;
    unsigned nexact;
};

// Front-to-back compositing of one queued survivor into this lane's pixel
// (rasterizer.cpp:88-100).  Branch-free: a lane that does not take the splat
// blends alpha = 0.
//
// CAREFUL = false is the speculative form the batch loop runs over a group of
// survivors: it only records in near_acc whether any FP32 value fell inside
// the guard band of a threshold; the group is then replayed from the saved
// pixel state with CAREFUL = true, which re-takes those decisions in FP64.
template <int FAM, bool CAREFUL>
__device__ __forceinline__ void fwd_visit(const KParams& kp, const float4* __restrict__ recs,
                                          const float4* __restrict__ qe, float fx, float fy,
                                          FwdPixel& px, bool& near_acc) {
    const float4 s0 = qe[0];
    const float4 s1 = qe[1];
    const float4 s2 = qe[2];
    const float dx = fx - s0.x, dy = fy - s0.y;
    const float m = quad_m(s0.z, s0.w, s1.x, dx, dy);
    const bool live = !(px.T < kTFloorF);
    bool hit, near;
    float a_raw, w, dwdm;
    fast_decide<FAM, false>(kp, m, s1.z, s1.y, hit, near, a_raw, w, dwdm);
    float alpha = fminf(kAlphaClampF, a_raw);
    if constexpr (CAREFUL) {
        if (kp.exact && near && live && __float_as_int(s2.w) >= 0) {
            const float4 r = exact_decide(kp, recs, __float_as_int(s2.w), fx, fy);
            hit = __float_as_int(r.w) & 1;
            alpha = r.x;
            ++px.nexact;
        }
    } else {
        near_acc = near_acc || near;
    }
    const float hitf = (hit && live) ? 1.f : 0.f;
    alpha *= hitf;
    // rasterizer.cpp:96-100
    const float at = alpha * px.T;
    px.cr = fmaf(s2.x, at, px.cr);
    px.cg = fmaf(s2.y, at, px.cg);
    px.cb = fmaf(s2.z, at, px.cb);
    const float Tn = fmaf(-alpha, px.T, px.T);
    px.contrib += hitf;
    // the step that crossed the floor (a live lane that does not take the splat keeps T)
    if (live && Tn < kTFloorF) px.proc = __float_as_int(s1.w) + 1;
    px.T = Tn;
}

template <int FAM>
__global__ void __launch_bounds__(kThreads, 3)
render_fwd_kernel(KParams kp, const float4* __restrict__ recs, const float4* __restrict__ stream,
                  size_t stream_stride, const int2* __restrict__ ranges,
                  const int* __restrict__ point_list, int W, int H, int tiles_x, float bg0,
                  float bg1, float bg2, float* __restrict__ image, float* __restrict__ t_final,
                  int* __restrict__ processed, int* __restrict__ contributors,
                  float4* __restrict__ surv, size_t surv_stride, int* __restrict__ surv_count,
                  unsigned long long* __restrict__ counters) {
    __shared__ float4 queue[kWarpsPerCta][kFwdQueueCap * 3];
    const int tile = blockIdx.x;
    // the warp index through a warp reduction: the compiler then knows it is warp-uniform and
    // keeps the block rectangle, queue pointer and loop control in uniform registers
    const int warp = __reduce_min_sync(kFull, (int)(threadIdx.x >> 5)), lane = threadIdx.x & 31;
    const int bx = (tile % tiles_x) * DARBS_TILE_SIZE + (warp & 1) * 8;
    const int by = (tile / tiles_x) * DARBS_TILE_SIZE + (warp >> 1) * 4;
    if (bx >= W || by >= H) return;  // whole block outside the image
    const int pxl = bx + (lane & 7), pyl = by + (lane >> 3);
    const bool inside = pxl < W && pyl < H;
    const float fx = pxl + 0.5f, fy = pyl + 0.5f;
    const float X0 = bx + 0.5f, X1 = bx + 7.5f, Y0 = by + 0.5f, Y1 = by + 3.5f;
    const int2 range = ranges[tile];
    const int beg = range.x, end = range.y;
    const float band2 = 2.f * kp.band;

    FwdPixel px;
    px.T = inside ? 1.f : 0.f;
    px.cr = px.cg = px.cb = 0.f;
    px.contrib = 0.f;
    px.proc = end - beg;
    px.nexact = 0;
    int nsurv = 0;
    float4* q = queue[warp];
    const unsigned lt_mask = (1u << lane) - 1u;
    int head = 0, qn = 0;  // ring: entries [head, head + qn)
    // this block's survivors, in queue format, kept for the backward pass (three arrays v0 | v1 | v2)
    float4* sl = surv + survivor_list_offset(beg, end, warp);

    // One register set holds the chunk under test and is reloaded with the next chunk as soon as
    // its entries have been queued, so the loads fly during the compositing below.
    Entry e;
    int idx = -1;
    load_entry(e, idx, stream, stream_stride, point_list, beg + lane, end);
    for (int base = beg; base < end; base += 32) {
        const int pos = base - beg + lane;
        const bool survive = base + lane < end && block_survives(e.v0.x, e.v0.y, e.v0.z, e.v0.w, e.v1.x, e.v1.w,
                                                                 e.v2.w, e.v1.z, band2, X0, X1, Y0, Y1);
        const unsigned mask = __ballot_sync(kFull, survive);
        if (survive) {
            const int rank = __popc(mask & lt_mask);
            queue_push<kFwdQueueCap>(q, head + qn + rank, e, pos, idx);
            float4* dst = sl + nsurv + rank;
            dst[0] = e.v0;
            dst[surv_stride] = make_float4(e.v1.x, e.v1.y, e.v1.z, __int_as_float(pos));
            dst[2 * surv_stride] = make_float4(e.v2.x, e.v2.y, e.v2.z, __int_as_float(idx));
        }
        const int cnt = __popc(mask);
        qn += cnt;
        nsurv += cnt;
        load_entry(e, idx, stream, stream_stride, point_list, base + 32 + lane, end);
        if (base + 32 >= end) qn = queue_pad<kFwdQueueCap, kGroup>(q, head, qn, lane);
        if (qn < kGroup) continue;
        __syncwarp();
        do {
            const float4* qb = q + head * 3;
            const FwdPixel save = px;
            bool near_acc = false;
#pragma unroll
            for (int j = 0; j < kGroup; ++j) fwd_visit<FAM, false>(kp, recs, qb + j * 3, fx, fy, px, near_acc);
            if (kp.exact && __any_sync(kFull, near_acc)) {  // a few groups per thousand
                px = save;
                for (int j = 0; j < kGroup; ++j) fwd_visit<FAM, true>(kp, recs, qb + j * 3, fx, fy, px, near_acc);
            }
            head = head + kGroup == kFwdQueueCap ? 0 : head + kGroup;
            qn -= kGroup;
        } while (qn >= kGroup);
        __syncwarp();
        if (!__any_sync(kFull, !(px.T < kTFloorF))) break;
    }
    // pixels whose transmittance came within the guard band of the floor: the last value
    // (the first below the floor, or the final one) and, for a pixel that crossed, the value
    // just before the crossing, recovered from the splat that crossed it
    unsigned nfloor = 0;
    if (inside) {
        nfloor = fabsf(px.T - kTFloorF) < 2e-9f;
        if (px.T < kTFloorF && px.proc > 0) {
            const int idx = __ldg(point_list + beg + px.proc - 1);
            const float4 v0 = __ldg(recs + kRecVecs * (int64_t)idx);
            const float4 v1 = __ldg(recs + kRecVecs * (int64_t)idx + 1);
            bool hit, near;
            float a_raw, w, dwdm;
            fast_decide<FAM, false>(kp, quad_m(v0.z, v0.w, v1.x, fx - v0.x, fy - v0.y), v1.z, v1.y, hit, near,
                                    a_raw, w, dwdm);
            const float t_cross = px.T / (1.0f - fminf(kAlphaClampF, a_raw));
            nfloor = nfloor || fabsf(t_cross - kTFloorF) < 4e-9f;
        }
        size_t p = (size_t)pyl * W + pxl;
        image[p * 3 + 0] = fmaf(bg0, px.T, px.cr);
        image[p * 3 + 1] = fmaf(bg1, px.T, px.cg);
        image[p * 3 + 2] = fmaf(bg2, px.T, px.cb);
        t_final[p] = px.T;
        processed[p] = px.proc;
        contributors[p] = (int)px.contrib;
    }
    // instrumentation: one atomic per warp per counter
    const unsigned nexact = __reduce_add_sync(kFull, px.nexact);
    nfloor = __reduce_add_sync(kFull, nfloor);
    if (lane == 0) {
        surv_count[tile * kWarpsPerCta + warp] = nsurv;
        atomicAdd(counters + CNT_SURVIVORS, (unsigned long long)nsurv);
        if (nexact) atomicAdd(counters + CNT_EXACT, (unsigned long long)nexact);
        if (nfloor) atomicAdd(counters + CNT_TFLOOR, (unsigned long long)nfloor);
    }
}

// ----------------------------------------------------------------- backward
//
// One CTA of 4 warps per HALF tile (16x8 pixels); a warp owns an 8x4 block as in
// the forward.  The list is walked back to front in two sweeps per batch of
// kBwdBatch queued survivors:
//   sweep 1 (lane = pixel): the reverse compositing chain of rasterizer.cpp:
//       189-213; per (pixel, survivor) it leaves three numbers in a padded
//       shared-memory matrix: wgt = alpha * T_before (colour gradient weight),
//       y = d_alpha * w (opacity gradient term), z = d_alpha * o * dw/dm (the
//       common factor of the conic and mean gradients), the last two gated by
//       the alpha clamp;
//   sweep 2 (lane = survivor x half of the pixels): each lane sums its
//       survivor's nine gradients over 16 pixels in registers; one shuffle
//       folds the two halves.  No per-survivor cross-lane reduction.
// Then one red.global.add per gradient component per survivor.
constexpr int kBwdWarps = 4;
constexpr int kBwdThreads = 32 * kBwdWarps;
constexpr int kBwdBatch = 16;
constexpr int kXStride = kBwdBatch + 1;  // odd: conflict-free both by row and by column
constexpr int kBwdQueueCap = 48;         // 32 appended per chunk on top of at most kBwdBatch - 1 left over
// per warp: queue, staging ring, 32 pixel gradients, three 32 x kXStride exchange matrices
constexpr int kSplatGradStride = 12;     // internal gradient rows are padded to 12 floats for 128-bit atomics

struct BwdPixel {
    float T;       // transmittance in front of the cursor
    float s;       // <g, colour composited behind the cursor> (rasterizer.cpp:180)
    float g0, g1, g2;
    int nproc;
    unsigned nexact;
};

template <int FAM, bool CAREFUL>
__device__ __forceinline__ void bwd_visit(const KParams& kp, const float4* __restrict__ recs,
                                          const float4* __restrict__ qe, float fx, float fy,
                                          BwdPixel& px, float* __restrict__ xw,
                                          float* __restrict__ xy, float* __restrict__ xz,
                                          bool& near_acc) {
    const float4 s0 = qe[0];
    const float4 s1 = qe[1];
    const float4 s2 = qe[2];
    const float dx = fx - s0.x, dy = fy - s0.y;
    const float m = quad_m(s0.z, s0.w, s1.x, dx, dy);
    const bool elig = __float_as_int(s1.w) < px.nproc;
    bool hit, near;
    float a_raw, w, dwdm;
    fast_decide<FAM, true>(kp, m, s1.z, s1.y, hit, near, a_raw, w, dwdm);
    float alpha = fminf(kAlphaClampF, a_raw);
    bool gate = a_raw < kAlphaClampF;
    if constexpr (CAREFUL) {
        if (kp.exact && near && elig && __float_as_int(s2.w) >= 0) {
            const float4 r = exact_decide(kp, recs, __float_as_int(s2.w), fx, fy);
            const int flags = __float_as_int(r.w);
            hit = flags & 1;
            gate = flags & 2;
            alpha = r.x;
            w = r.y;
            dwdm = r.z;
            ++px.nexact;
        }
    } else {
        near_acc = near_acc || near;
    }
    hit = hit && elig;
    gate = gate && hit;
    alpha = hit ? alpha : 0.f;
    // rasterizer.cpp:189-213 with s = <g, accum_behind>
    const float om = 1.0f - alpha;
    const float rc = rcp_approx(om);
    const float t_before = px.T * rc;
    const float wgt = alpha * t_before;
    const float gc = fmaf(px.g2, s2.z, fmaf(px.g1, s2.y, px.g0 * s2.x));
    const float d_alpha = fmaf(t_before, gc, -(rc * px.s));
    const float da = gate ? d_alpha : 0.f;
    *xw = wgt;
    *xy = da * w;
    *xz = da * s1.y * dwdm;
    px.s = fmaf(gc, wgt, px.s);
    if (hit) px.T = t_before;
}

template <int FAM>
__global__ void __launch_bounds__(kBwdThreads, 4)
render_bwd_kernel(KParams kp, const float4* __restrict__ recs, const int2* __restrict__ ranges,
                  const float4* __restrict__ surv, size_t surv_stride,
                  const int* __restrict__ surv_count, int W, int H, int tiles_x, float bg0, float bg1,
                  float bg2, const float* __restrict__ grad_image,
                  const float* __restrict__ t_final, const int* __restrict__ processed,
                  float* __restrict__ grads, unsigned long long* __restrict__ counters) {
    __shared__ float4 queue[kBwdWarps][kBwdQueueCap * 3];
    __shared__ float xch[kBwdWarps][3][32 * kXStride];
    __shared__ float4 gpix[kBwdWarps][32];
    const int tile = blockIdx.x >> 1, half = blockIdx.x & 1;
    const int warp = __reduce_min_sync(kFull, (int)(threadIdx.x >> 5)), lane = threadIdx.x & 31;
    const int blk = half * kBwdWarps + warp;  // the forward's warp index of this block
    const int bx = (tile % tiles_x) * DARBS_TILE_SIZE + (warp & 1) * 8;
    const int by = (tile / tiles_x) * DARBS_TILE_SIZE + half * 8 + (warp >> 1) * 4;
    if (bx >= W || by >= H) return;
    const int pxl = bx + (lane & 7), pyl = by + (lane >> 3);
    const bool inside = pxl < W && pyl < H;
    const float fx = pxl + 0.5f, fy = pyl + 0.5f;
    const float X0 = bx + 0.5f, Y0 = by + 0.5f;
    const int2 range = ranges[tile];

    BwdPixel px;
    px.g0 = px.g1 = px.g2 = 0.f;
    px.T = 1.f;
    px.nproc = 0;
    px.nexact = 0;
    if (inside) {
        size_t p = (size_t)pyl * W + pxl;
        px.g0 = grad_image[p * 3 + 0];
        px.g1 = grad_image[p * 3 + 1];
        px.g2 = grad_image[p * 3 + 2];
        px.T = t_final[p];
        px.nproc = processed[p];
    }
    const int wmax = __reduce_max_sync(kFull, px.nproc);
    if (wmax == 0) return;
    px.s = (px.g0 * bg0 + px.g1 * bg1 + px.g2 * bg2) * px.T;

    float4* q = queue[warp];
    float4* gp = gpix[warp];
    float* xw = xch[warp][0];
    float* xy = xch[warp][1];
    float* xz = xch[warp][2];
    gp[lane] = make_float4(px.g0, px.g1, px.g2, 0.f);
    const unsigned lt_mask = (1u << lane) - 1u;
    int head = 0, qn = 0;

    // sweep-2 role of this lane: survivor sj of the batch, pixels [16 sh, 16 sh + 16)
    const int sj = lane & (kBwdBatch - 1), sh = lane >> 4;
    const float* rw = xw + (sh * 16) * kXStride + sj;
    const float* ry = xy + (sh * 16) * kXStride + sj;
    const float* rz = xz + (sh * 16) * kXStride + sj;
    const float4* rg = gp + sh * 16;
    const float ex0 = X0, ey0 = Y0 + 2.f * sh;

    // The block's survivors, in the queue format the forward left them in, walked from the
    // back: lane l of a chunk takes the l-th entry from the chunk's end, so lane order is
    // descending list position and the loads are contiguous.  Entries the forward queued beyond
    // the last position any of this block's pixels processed are dropped here.
    const float4* sl = surv + survivor_list_offset(range.x, range.y, blk);
    const int nsl = surv_count[tile * kWarpsPerCta + blk];
    auto load_surv = [&](Entry& e, int k) {
        if (k >= 0) {
            e.v0 = __ldg(sl + k);
            e.v1 = __ldg(sl + surv_stride + k);
            e.v2 = __ldg(sl + 2 * surv_stride + k);
        }
    };
    Entry e;
    load_surv(e, nsl - 1 - lane);
    for (int top = nsl; top > 0; top -= 32) {
        const bool survive = top - 1 - lane >= 0 && __float_as_int(e.v1.w) < wmax;
        const unsigned mask = __ballot_sync(kFull, survive);
        if (survive) {
            int slot = head + qn + __popc(mask & lt_mask);
            if (slot >= kBwdQueueCap) slot -= kBwdQueueCap;
            q[slot * 3 + 0] = e.v0;
            q[slot * 3 + 1] = e.v1;
            q[slot * 3 + 2] = e.v2;
        }
        qn += __popc(mask);
        load_surv(e, top - 33 - lane);
        if (top <= 32) qn = queue_pad<kBwdQueueCap, kBwdBatch>(q, head, qn, lane);
        while (qn >= kBwdBatch) {
            const float4* qb = q + head * 3;
            __syncwarp();
            // ---- sweep 1: lane = pixel
            float* ww = xw + lane * kXStride;
            float* wy = xy + lane * kXStride;
            float* wz = xz + lane * kXStride;
            for (int j0 = 0; j0 < kBwdBatch; j0 += kGroup) {
                const BwdPixel save = px;
                bool near_acc = false;
#pragma unroll
                for (int j = 0; j < kGroup; ++j)
                    bwd_visit<FAM, false>(kp, recs, qb + (j0 + j) * 3, fx, fy, px, ww + j0 + j, wy + j0 + j,
                                          wz + j0 + j, near_acc);
                if (kp.exact && __any_sync(kFull, near_acc)) {  // a few groups per thousand
                    px = save;
                    for (int j = 0; j < kGroup; ++j)
                        bwd_visit<FAM, true>(kp, recs, qb + (j0 + j) * 3, fx, fy, px, ww + j0 + j, wy + j0 + j,
                                             wz + j0 + j, near_acc);
                }
            }
            __syncwarp();
            // ---- sweep 2: lane = (survivor, half of the pixels)
            {
                const float4 r0 = qb[sj * 3 + 0];
                const float4 r1 = qb[sj * 3 + 1];
                const float4 r2 = qb[sj * 3 + 2];
                const float ex = ex0 - r0.x, ey = ey0 - r0.y;
                float dc0 = 0.f, dc1 = 0.f, dc2 = 0.f, dop = 0.f, wsum = 0.f;
                float sxx = 0.f, sxy = 0.f, syy = 0.f, sx = 0.f, sy = 0.f;
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const float wv = rw[i * kXStride];
                    const float yv = ry[i * kXStride];
                    const float zv = rz[i * kXStride];
                    const float4 g = rg[i];
                    const float dx = ex + (float)(i & 7), dy = ey + (float)(i >> 3);
                    dc0 = fmaf(g.x, wv, dc0);
                    dc1 = fmaf(g.y, wv, dc1);
                    dc2 = fmaf(g.z, wv, dc2);
                    wsum += wv;
                    dop += yv;
                    const float zx = zv * dx, zy = zv * dy;
                    sxx = fmaf(zx, dx, sxx);
                    sxy = fmaf(zx, dy, sxy);
                    syy = fmaf(zy, dy, syy);
                    sx += zx;
                    sy += zy;
                }
                // fold the two pixel halves (lanes l and l ^ 16 hold the same survivor)
                dc0 += __shfl_xor_sync(kFull, dc0, 16);
                dc1 += __shfl_xor_sync(kFull, dc1, 16);
                dc2 += __shfl_xor_sync(kFull, dc2, 16);
                dop += __shfl_xor_sync(kFull, dop, 16);
                wsum += __shfl_xor_sync(kFull, wsum, 16);
                sxx += __shfl_xor_sync(kFull, sxx, 16);
                sxy += __shfl_xor_sync(kFull, sxy, 16);
                syy += __shfl_xor_sync(kFull, syy, 16);
                sx += __shfl_xor_sync(kFull, sx, 16);
                sy += __shfl_xor_sync(kFull, sy, 16);
                if (sh == 0 && wsum > 0.f) {
                    // SplatGrads order d_color[3], d_opacity, d_conic_a, d_conic_b, d_conic_c, d_mu2;
                    // m = scale * (a dx^2 + 2 b dx dy + c dy^2): dm/da = scale dx^2, dm/db = 2 scale dx dy,
                    // dm/d mu = -(2A dx + B dy, B dx + 2C dy) with (A, B, C) the scaled record values.
                    float* dst = grads + (size_t)__float_as_int(r2.w) * kSplatGradStride;
                    atomicAdd(reinterpret_cast<float4*>(dst), make_float4(dc0, dc1, dc2, dop));
                    atomicAdd(reinterpret_cast<float4*>(dst) + 1,
                              make_float4(kp.scale * sxx, 2.f * kp.scale * sxy, kp.scale * syy,
                                          -fmaf(2.f * r0.z, sx, r0.w * sy)));
                    atomicAdd(dst + 8, -fmaf(r0.w, sx, 2.f * r1.x * sy));
                }
            }
            head = head + kBwdBatch == kBwdQueueCap ? 0 : head + kBwdBatch;
            qn -= kBwdBatch;
        }
    }
    const unsigned nexact = __reduce_add_sync(kFull, px.nexact);
    if (lane == 0 && nexact) atomicAdd(counters + CNT_EXACT, (unsigned long long)nexact);
}

__global__ void export_grads_kernel(int64_t count, const float* __restrict__ padded, float* __restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= count) return;
    out[i] = padded[(i / DARBS_GRADS_PER_SPLAT) * kSplatGradStride + i % DARBS_GRADS_PER_SPLAT];
}

// ------------------------------------------------------------- eval (tests)
template <int FAM>
__device__ void eval_one_fast(const KParams& kp, float dm2, float& w, float& dw) {
    if constexpr (FAM == FAM_GENERIC) {
        generic_eval(kp, dm2, w, dw);
    } else {
        float m = kp.scale * dm2, dwdm;
        fam_eval<FAM>(m, w, dwdm);
        dw = dwdm * kp.scale;
    }
}

__global__ void eval_kernel(KParams kp, int64_t n, const float* __restrict__ dm2,
                            float* __restrict__ w, float* __restrict__ dw, int exact) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    float x = dm2[i];
    float wo = 0.f, dwo = 0.f;
    bool past = kp.unbounded ? x > kp.cutoff : x >= kp.cutoff;  // kernel.cpp:136
    if (exact) {
        double wd, dwd;
        eval_exact(kp, (double)x, wd, dwd);
        wo = (float)wd;
        dwo = (float)dwd;
    } else if (!past) {
        switch (kp.fam) {
            case FAM_GAUSS2: eval_one_fast<FAM_GAUSS2>(kp, x, wo, dwo); break;
            case FAM_HCOS2: eval_one_fast<FAM_HCOS2>(kp, x, wo, dwo); break;
            case FAM_RCOS1: eval_one_fast<FAM_RCOS1>(kp, x, wo, dwo); break;
            case FAM_IMQ: eval_one_fast<FAM_IMQ>(kp, x, wo, dwo); break;
            default: eval_one_fast<FAM_GENERIC>(kp, x, wo, dwo); break;
        }
    }
    if (w) w[i] = wo;
    if (dw) dw[i] = dwo;
}

// ------------------------------------------------- work counters (V and C)
__global__ void sum_counts_kernel(int64_t px, const int* __restrict__ processed,
                                  const int* __restrict__ contributors,
                                  unsigned long long* __restrict__ counters) {
    unsigned long long v = 0, c = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < px;
         i += (int64_t)gridDim.x * blockDim.x) {
        v += (unsigned)processed[i];
        c += (unsigned)contributors[i];
    }
    for (int o = 16; o > 0; o >>= 1) {
        v += __shfl_xor_sync(kFull, v, o);
        c += __shfl_xor_sync(kFull, c, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(counters + 1, v);
        atomicAdd(counters + 2, c);
    }
}

}  // namespace

// ---------------------------------------------------------------- launchers
darbs_status launch_pack(darbs_cuda_ctx* ctx, const KParams& kp, int64_t n, const float* mu2,
                         const float* conic, const float* opacity, const float* rgb) {
    DARBS_TRY(reserve(ctx, ctx->recs, sizeof(float4) * kRecVecs * (size_t)(n > 0 ? n : 1)));
    if (n == 0) return DARBS_OK;
    int threads = 256;
    int64_t blocks = (n + threads - 1) / threads;
    pack_kernel<<<(unsigned)blocks, threads, 0, ctx->stream>>>(kp, n, mu2, conic, opacity, rgb,
                                                               (float4*)ctx->recs.ptr);
    return check_launch(ctx, "pack_kernel");
}

// Copies the records of the K sorted list entries into list order (see load_entry).
darbs_status launch_gather(darbs_cuda_ctx* ctx) {
    const int64_t k = ctx->fwd_entries;
    DARBS_TRY(reserve(ctx, ctx->stream_recs, sizeof(float4) * 3 * (size_t)(k > 0 ? k : 1)));
    if (k == 0) return DARBS_OK;
    gather_kernel<<<(unsigned)((k + 255) / 256), 256, 0, ctx->stream>>>(
        k, point_list_ptr(ctx), (const float4*)ctx->recs.ptr, (float4*)ctx->stream_recs.ptr);
    return check_launch(ctx, "gather_kernel");
}

darbs_status launch_render_fwd(darbs_cuda_ctx* ctx, const KParams& kp, int width, int height,
                               const float bg[3], float* image, float* t_final,
                               int32_t* processed, int32_t* contributors) {
    int tiles = ctx->tiles_x * ctx->tiles_y;
    if (tiles == 0) return DARBS_OK;
    // per-block survivor streams for the backward pass: 8 regions per tile, each as long as the
    // tile's list (address space only; the forward writes survivors, a quarter of it or less)
    const size_t k = (size_t)(ctx->fwd_entries > 0 ? ctx->fwd_entries : 1);
    const size_t surv_stride = kWarpsPerCta * k;
    DARBS_TRY(reserve(ctx, ctx->surv, sizeof(float4) * 3 * surv_stride));
    DARBS_TRY(reserve(ctx, ctx->surv_count, sizeof(int) * kWarpsPerCta * (size_t)tiles));
    ctx->surv_stride = (int64_t)surv_stride;
    auto* counters = (unsigned long long*)ctx->counters.ptr;
    const float4* recs = (const float4*)ctx->recs.ptr;
    const int2* ranges = (const int2*)ctx->ranges.ptr;
    const int* plist = point_list_ptr(ctx);
#define DARBS_LAUNCH_FWD(F)                                                                       \
    render_fwd_kernel<F><<<tiles, kThreads, 0, ctx->stream>>>(                                    \
        kp, recs, (const float4*)ctx->stream_recs.ptr, k, ranges, plist, width, height,           \
        ctx->tiles_x, bg[0], bg[1], bg[2], image, t_final, processed, contributors,               \
        (float4*)ctx->surv.ptr, surv_stride, (int*)ctx->surv_count.ptr, counters)
    switch (kp.fam) {
        case FAM_GAUSS2: DARBS_LAUNCH_FWD(FAM_GAUSS2); break;
        case FAM_HCOS2: DARBS_LAUNCH_FWD(FAM_HCOS2); break;
        case FAM_RCOS1: DARBS_LAUNCH_FWD(FAM_RCOS1); break;
        case FAM_IMQ: DARBS_LAUNCH_FWD(FAM_IMQ); break;
        default: DARBS_LAUNCH_FWD(FAM_GENERIC); break;
    }
#undef DARBS_LAUNCH_FWD
    return check_launch(ctx, "render_fwd_kernel");
}

// Accumulates into ctx->splat_grads, n rows of kSplatGradStride floats (SplatGrads order in the
// first nine), zeroed here.
darbs_status launch_render_bwd(darbs_cuda_ctx* ctx, const KParams& kp, int width, int height,
                               const float bg[3], const float* grad_image, const float* t_final,
                               const int32_t* processed, int64_t n) {
    const size_t bytes = sizeof(float) * kSplatGradStride * (size_t)(n > 0 ? n : 1);
    DARBS_TRY(reserve(ctx, ctx->splat_grads, bytes));
    DARBS_CUDA_TRY(ctx, cudaMemsetAsync(ctx->splat_grads.ptr, 0, bytes, ctx->stream));
    int tiles = ctx->tiles_x * ctx->tiles_y;
    if (tiles == 0 || n == 0) return DARBS_OK;
    auto* counters = (unsigned long long*)ctx->counters.ptr;
    const float4* recs = (const float4*)ctx->recs.ptr;
    const int2* ranges = (const int2*)ctx->ranges.ptr;
#define DARBS_LAUNCH_BWD(F)                                                                       \
    render_bwd_kernel<F><<<2 * tiles, kBwdThreads, 0, ctx->stream>>>(                             \
        kp, recs, ranges, (const float4*)ctx->surv.ptr, (size_t)ctx->surv_stride,                 \
        (const int*)ctx->surv_count.ptr, width, height, ctx->tiles_x, bg[0], bg[1], bg[2],        \
        grad_image, t_final, processed, (float*)ctx->splat_grads.ptr, counters)
    switch (kp.fam) {
        case FAM_GAUSS2: DARBS_LAUNCH_BWD(FAM_GAUSS2); break;
        case FAM_HCOS2: DARBS_LAUNCH_BWD(FAM_HCOS2); break;
        case FAM_RCOS1: DARBS_LAUNCH_BWD(FAM_RCOS1); break;
        case FAM_IMQ: DARBS_LAUNCH_BWD(FAM_IMQ); break;
        default: DARBS_LAUNCH_BWD(FAM_GENERIC); break;
    }
#undef DARBS_LAUNCH_BWD
    return check_launch(ctx, "render_bwd_kernel");
}

// ctx->splat_grads (padded rows) -> out[9 n], the SplatGrads layout of the ABI.
darbs_status launch_export_grads(darbs_cuda_ctx* ctx, int64_t n, float* out) {
    if (n == 0) return DARBS_OK;
    const int64_t count = n * DARBS_GRADS_PER_SPLAT;
    export_grads_kernel<<<(unsigned)((count + 255) / 256), 256, 0, ctx->stream>>>(
        count, (const float*)ctx->splat_grads.ptr, out);
    return check_launch(ctx, "export_grads_kernel");
}

darbs_status launch_eval(darbs_cuda_ctx* ctx, const KParams& kp, int64_t n, const float* dm2,
                         float* w, float* dw, int exact) {
    if (n == 0) return DARBS_OK;
    int threads = 256;
    int64_t blocks = (n + threads - 1) / threads;
    eval_kernel<<<(unsigned)blocks, threads, 0, ctx->stream>>>(kp, n, dm2, w, dw, exact);
    return check_launch(ctx, "eval_kernel");
}

darbs_status launch_sum_counts(darbs_cuda_ctx* ctx, int64_t px, const int32_t* processed,
                               const int32_t* contributors) {
    if (px == 0) return DARBS_OK;
    sum_counts_kernel<<<148 * 4, 256, 0, ctx->stream>>>(px, processed, contributors,
                                                        (unsigned long long*)ctx->counters.ptr);
    return check_launch(ctx, "sum_counts_kernel");
}

}  // namespace darbs_b200
