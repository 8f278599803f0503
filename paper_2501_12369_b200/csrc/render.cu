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
    r[1] = make_float4(kp.scale * c, o, thr_m, 0.f);
    r[2] = make_float4(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2], 0.f);
    r[3] = make_float4(a, b, c, 0.f);
}

// ------------------------------------------------------------ shared pieces

// Lower bound of m(d) = A dx^2 + B dx dy + C dy^2 over the rectangle of pixel
// centres [X0,X1]x[Y0,Y1] (d measured from the splat centre).  A, C > 0 and
// 4AC > B^2 (the pack kernel sends every other conic down the NaN path).  The
// minimum of a convex quadratic over a box that does not contain the
// unconstrained minimiser lies on an edge facing it.
__device__ __forceinline__ bool block_survives(float mx, float my, float A, float B, float C,
                                               float thr, float band, float X0, float X1,
                                               float Y0, float Y1) {
    if (!(thr == thr)) return true;  // NaN threshold: always decided in FP64
    float ex0 = X0 - mx, ex1 = X1 - mx, ey0 = Y0 - my, ey1 = Y1 - my;
    bool out_x = (ex0 > 0.f) || (ex1 < 0.f);
    bool out_y = (ey0 > 0.f) || (ey1 < 0.f);
    float mmin = 0.f;
    if (out_x || out_y) {
        mmin = 3.0e38f;
        if (out_x) {
            float dx = ex0 > 0.f ? ex0 : ex1;
            float dy = __fdividef(-0.5f * B * dx, C);
            dy = fminf(fmaxf(dy, ey0), ey1);
            mmin = fmaf(fmaf(A, dx, B * dy), dx, C * dy * dy);
        }
        if (out_y) {
            float dy = ey0 > 0.f ? ey0 : ey1;
            float dx = __fdividef(-0.5f * B * dy, A);
            dx = fminf(fmaxf(dx, ex0), ex1);
            mmin = fminf(mmin, fmaf(fmaf(A, dx, B * dy), dx, C * dy * dy));
        }
    }
    // Per-pixel decisions can only be positive for m <= thr + band; keep a
    // relative margin for the FP32 rounding of mmin itself.
    return mmin * 0.9999f <= thr + 2.f * band;
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

struct Decision {
    float alpha;  // clamped alpha actually blended
    float w;      // kernel weight
    float dwdm;   // d weight / d m
    bool gate;    // alpha_raw < 0.99: the clamp lets the gradient through (rasterizer.cpp:202)
};

// The reference's per-visit logic (rasterizer.cpp:90-95 / :181-187) in FP64 on
// the values the reference would see (the float32 inputs widened), with its
// expression order (conic_dm2 rasterizer.cpp:19-21).
__device__ __noinline__ bool exact_decide(const KParams& kp, const float4* __restrict__ recs,
                                          int idx, float fx, float fy, Decision& out) {
    const float4 v0 = __ldg(recs + kRecVecs * (int64_t)idx);
    const float4 v1 = __ldg(recs + kRecVecs * (int64_t)idx + 1);
    const float4 v3 = __ldg(recs + kRecVecs * (int64_t)idx + 3);
    double dx = (double)fx - (double)v0.x, dy = (double)fy - (double)v0.y;
    double a = v3.x, b = v3.y, c = v3.z, o = v1.y;
    double dm2 = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(a, dx), dx),
                                     __dmul_rn(__dmul_rn(__dmul_rn(2.0, b), dx), dy)),
                           __dmul_rn(__dmul_rn(c, dy), dy));
    if (!(dm2 >= 0.0)) return false;  // dm2 < 0 (or NaN, which the reference rejects)
    double w, dw;
    eval_exact(kp, dm2, w, dw);
    double alpha_raw = o * w;
    double alpha = fmin(kAlphaClampD, alpha_raw);
    if (alpha < kAlphaSkipD) return false;
    out.alpha = (float)alpha;
    out.w = (float)w;
    out.dwdm = (float)(dw / (double)kp.scale);
    out.gate = alpha_raw < kAlphaClampD;
    return true;
}

// One (pixel, entry) visit.  m = scaled squared Mahalanobis distance computed
// by the caller with a fixed FMA order shared by forward and backward, so both
// passes take identical decisions.
template <int FAM, bool GRAD>
__device__ __forceinline__ bool visit(const KParams& kp, const float4* __restrict__ recs, int idx,
                                      float fx, float fy, float m, float thr, float o,
                                      Decision& dec, unsigned& nexact) {
    bool near;
    if constexpr (FAM == FAM_GENERIC) {
        // m == dm2 here (scale 1); thr == cutoff.
        near = !(fabsf(m) > kp.band) || !(fabsf(m - kp.cutoff) > kp.band);
        if (!near) {
            if (m < 0.f || m > kp.cutoff) return false;
            generic_eval(kp, m, dec.w, dec.dwdm);
            float alpha_raw = o * dec.w;
            near = !(fabsf(alpha_raw - kAlphaSkipF) > 2e-6f);
            if (GRAD) near = near || !(fabsf(alpha_raw - kAlphaClampF) > 2e-6f);
            if (!near || !kp.exact) {
                dec.alpha = fminf(kAlphaClampF, alpha_raw);
                dec.gate = alpha_raw < kAlphaClampF;
                return !(dec.alpha < kAlphaSkipF);
            }
        }
        if (!kp.exact) return false;
    } else {
        float d = thr - m;
        near = !(fabsf(d) > kp.band);  // also true for a NaN threshold
        if (!near || !kp.exact) {
            if (!(d > 0.f)) return false;
            if (GRAD) {
                fam_eval<FAM>(m, dec.w, dec.dwdm);
            } else {
                dec.w = fam_weight<FAM>(m);
            }
            float alpha_raw = o * dec.w;
            dec.alpha = fminf(kAlphaClampF, alpha_raw);
            dec.gate = alpha_raw < kAlphaClampF;
            if (!GRAD || !kp.exact || fabsf(alpha_raw - kAlphaClampF) > 2e-6f) return true;
        }
    }
    ++nexact;
    return exact_decide(kp, recs, idx, fx, fy, dec);
}

__device__ __forceinline__ float quad_m(float A, float B, float C, float dx, float dy) {
    return fmaf(fmaf(A, dx, B * dy), dx, (C * dy) * dy);
}

struct Chunk {
    int idx;
    float4 v0, v1, v2;
};

__device__ __forceinline__ void load_chunk(Chunk& ch, const int* __restrict__ point_list,
                                           const float4* __restrict__ recs, int k, int end) {
    if (k < end) {
        ch.idx = __ldg(point_list + k);
        const float4* r = recs + kRecVecs * (int64_t)ch.idx;
        ch.v0 = __ldg(r);
        ch.v1 = __ldg(r + 1);
        ch.v2 = __ldg(r + 2);
    } else {
        ch.idx = -1;
    }
}

// ------------------------------------------------------------------ forward
template <int FAM>
__global__ void __launch_bounds__(kThreads)
render_fwd_kernel(KParams kp, const float4* __restrict__ recs, const int2* __restrict__ ranges,
                  const int* __restrict__ point_list, int W, int H, int tiles_x, float bg0,
                  float bg1, float bg2, float* __restrict__ image, float* __restrict__ t_final,
                  int* __restrict__ processed, int* __restrict__ contributors,
                  unsigned long long* __restrict__ counters) {
    __shared__ float4 stage[kWarpsPerCta][32 * 3];
    const int tile = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int bx = (tile % tiles_x) * DARBS_TILE_SIZE + (warp & 1) * 8;
    const int by = (tile / tiles_x) * DARBS_TILE_SIZE + (warp >> 1) * 4;
    if (bx >= W || by >= H) return;  // whole block outside the image
    const int px = bx + (lane & 7), py = by + (lane >> 3);
    const bool inside = px < W && py < H;
    const float fx = px + 0.5f, fy = py + 0.5f;
    const float X0 = bx + 0.5f, X1 = bx + 7.5f, Y0 = by + 0.5f, Y1 = by + 3.5f;
    const int2 range = ranges[tile];
    const int beg = range.x, end = range.y;

    float T = 1.f, cr = 0.f, cg = 0.f, cb = 0.f;
    int contrib = 0, proc = end - beg;
    bool active = inside;
    unsigned nexact = 0, nsurv = 0, nfloor = 0;
    float4* st = stage[warp];
    const unsigned lt_mask = (1u << lane) - 1u;

    Chunk cur, nxt;
    load_chunk(cur, point_list, recs, beg + lane, end);
    for (int base = beg; base < end; base += 32) {
        if (base + 32 < end) load_chunk(nxt, point_list, recs, base + 32 + lane, end);
        bool survive = cur.idx >= 0 &&
                       block_survives(cur.v0.x, cur.v0.y, cur.v0.z, cur.v0.w, cur.v1.x, cur.v1.z,
                                      kp.band, X0, X1, Y0, Y1);
        const unsigned mask = __ballot_sync(kFull, survive);
        const int cnt = __popc(mask);
        if (cnt) {
            if (survive) {
                int slot = __popc(mask & lt_mask);
                st[slot * 3 + 0] = cur.v0;
                st[slot * 3 + 1] = make_float4(cur.v1.x, cur.v1.y, cur.v1.z,
                                               __int_as_float(base - beg + lane));
                st[slot * 3 + 2] = make_float4(cur.v2.x, cur.v2.y, cur.v2.z,
                                               __int_as_float(cur.idx));
            }
            __syncwarp();
            nsurv += cnt;
            for (int j = 0; j < cnt; ++j) {
                const float4 s0 = st[j * 3 + 0];
                const float4 s1 = st[j * 3 + 1];
                if (active) {
                    float dx = fx - s0.x, dy = fy - s0.y;
                    float m = quad_m(s0.z, s0.w, s1.x, dx, dy);
                    Decision dec;
                    const float4 s2 = st[j * 3 + 2];
                    if (visit<FAM, false>(kp, recs, __float_as_int(s2.w), fx, fy, m, s1.z, s1.y,
                                          dec, nexact)) {
                        // rasterizer.cpp:96-100
                        float at = dec.alpha * T;
                        cr = fmaf(s2.x, at, cr);
                        cg = fmaf(s2.y, at, cg);
                        cb = fmaf(s2.z, at, cb);
                        T *= 1.0f - dec.alpha;
                        ++contrib;
                        if (fabsf(T - kTFloorF) < 2e-9f) ++nfloor;
                        if (T < kTFloorF) {
                            active = false;
                            proc = __float_as_int(s1.w) + 1;
                        }
                    }
                }
            }
            __syncwarp();
            if (!__any_sync(kFull, active)) break;
        }
        cur = nxt;
    }
    if (inside) {
        size_t p = (size_t)py * W + px;
        image[p * 3 + 0] = fmaf(bg0, T, cr);
        image[p * 3 + 1] = fmaf(bg1, T, cg);
        image[p * 3 + 2] = fmaf(bg2, T, cb);
        t_final[p] = T;
        processed[p] = proc;
        contributors[p] = contrib;
    }
    // instrumentation: one atomic per warp per counter
    nexact = __reduce_add_sync(kFull, nexact);
    nfloor = __reduce_add_sync(kFull, nfloor);
    if (lane == 0) {
        atomicAdd(counters + CNT_SURVIVORS, (unsigned long long)nsurv);
        if (nexact) atomicAdd(counters + CNT_EXACT, (unsigned long long)nexact);
        if (nfloor) atomicAdd(counters + CNT_TFLOOR, (unsigned long long)nfloor);
    }
}

// ----------------------------------------------------------------- backward

// Sum over the warp of 9 per-lane values; afterwards lanes 0,4,..,28 hold
// v[0..7] (lane >> 2) and every lane holds v[8] in `e`.  Reduce-scatter
// butterfly: 4+2+1 exchanges split the 8 values across lane bits 4,3,2, two
// more finish them; 14 shuffles instead of 45.
__device__ __forceinline__ float warp_reduce9(float (&v)[8], float& e, int lane) {
    const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
    float u[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float keep = h16 ? v[i + 4] : v[i];
        float send = h16 ? v[i] : v[i + 4];
        u[i] = keep + __shfl_xor_sync(kFull, send, 16);
    }
    float t[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        float keep = h8 ? u[i + 2] : u[i];
        float send = h8 ? u[i] : u[i + 2];
        t[i] = keep + __shfl_xor_sync(kFull, send, 8);
    }
    float keep = h4 ? t[1] : t[0];
    float send = h4 ? t[0] : t[1];
    float s = keep + __shfl_xor_sync(kFull, send, 4);
    s += __shfl_xor_sync(kFull, s, 2);
    s += __shfl_xor_sync(kFull, s, 1);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(kFull, e, o);
    return s;  // value index (lane >> 2) & 7 ... see caller
}

template <int FAM>
__global__ void __launch_bounds__(kThreads)
render_bwd_kernel(KParams kp, const float4* __restrict__ recs, const int2* __restrict__ ranges,
                  const int* __restrict__ point_list, int W, int H, int tiles_x, float bg0,
                  float bg1, float bg2, const float* __restrict__ grad_image,
                  const float* __restrict__ t_final, const int* __restrict__ processed,
                  float* __restrict__ grads, unsigned long long* __restrict__ counters) {
    __shared__ float4 stage[kWarpsPerCta][32 * 3];
    const int tile = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int bx = (tile % tiles_x) * DARBS_TILE_SIZE + (warp & 1) * 8;
    const int by = (tile / tiles_x) * DARBS_TILE_SIZE + (warp >> 1) * 4;
    if (bx >= W || by >= H) return;
    const int px = bx + (lane & 7), py = by + (lane >> 3);
    const bool inside = px < W && py < H;
    const float fx = px + 0.5f, fy = py + 0.5f;
    const float X0 = bx + 0.5f, X1 = bx + 7.5f, Y0 = by + 0.5f, Y1 = by + 3.5f;
    const int beg = ranges[tile].x;

    float g0 = 0.f, g1 = 0.f, g2 = 0.f, T = 1.f;
    int nproc = 0;
    if (inside) {
        size_t p = (size_t)py * W + px;
        g0 = grad_image[p * 3 + 0];
        g1 = grad_image[p * 3 + 1];
        g2 = grad_image[p * 3 + 2];
        T = t_final[p];
        nproc = processed[p];
    }
    const int wmax = __reduce_max_sync(kFull, nproc);
    if (wmax == 0) return;
    const int end = beg + wmax;
    // colour composited behind the cursor (rasterizer.cpp:180)
    float b0 = bg0 * T, b1 = bg1 * T, b2 = bg2 * T;

    // which of the 8 scatter-reduced values this lane owns, and its unscaling:
    // SplatGrads order d_color[3], d_opacity, d_conic_a, d_conic_b, d_conic_c, d_mu2.x
    // with m = scale*(a dx^2 + 2b dx dy + c dy^2): d/da = scale*dx^2, d/db = 2*scale*dx*dy.
    const int vi = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
    const float vmul = (vi == 4 || vi == 6) ? kp.scale : (vi == 5 ? 2.f * kp.scale : 1.f);
    const bool owner = (lane & 3) == 0;

    unsigned nexact = 0;
    float4* st = stage[warp];
    const unsigned gt_mask = lane == 31 ? 0u : ~((2u << lane) - 1u);

    const int nchunks = (wmax + 31) >> 5;
    Chunk cur, nxt;
    load_chunk(cur, point_list, recs, beg + (nchunks - 1) * 32 + lane, end);
    for (int ch = nchunks - 1; ch >= 0; --ch) {
        const int base = beg + ch * 32;
        if (ch > 0) load_chunk(nxt, point_list, recs, base - 32 + lane, end);
        bool survive = cur.idx >= 0 &&
                       block_survives(cur.v0.x, cur.v0.y, cur.v0.z, cur.v0.w, cur.v1.x, cur.v1.z,
                                      kp.band, X0, X1, Y0, Y1);
        const unsigned mask = __ballot_sync(kFull, survive);
        const int cnt = __popc(mask);
        if (cnt) {
            if (survive) {
                int slot = __popc(mask & gt_mask);  // descending list position
                st[slot * 3 + 0] = cur.v0;
                st[slot * 3 + 1] = make_float4(cur.v1.x, cur.v1.y, cur.v1.z,
                                               __int_as_float(base - beg + lane));
                st[slot * 3 + 2] = make_float4(cur.v2.x, cur.v2.y, cur.v2.z,
                                               __int_as_float(cur.idx));
            }
            __syncwarp();
            for (int j = 0; j < cnt; ++j) {
                const float4 s0 = st[j * 3 + 0];
                const float4 s1 = st[j * 3 + 1];
                const float4 s2 = st[j * 3 + 2];
                const int idx = __float_as_int(s2.w);
                float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                float e = 0.f;
                bool hit = false;
                if (__float_as_int(s1.w) < nproc) {
                    float dx = fx - s0.x, dy = fy - s0.y;
                    float m = quad_m(s0.z, s0.w, s1.x, dx, dy);
                    Decision dec;
                    hit = visit<FAM, true>(kp, recs, idx, fx, fy, m, s1.z, s1.y, dec, nexact);
                    if (hit) {
                        // rasterizer.cpp:189-213
                        float om = 1.0f - dec.alpha;
                        float rc = __frcp_rn(om);
                        float t_before = T * rc;
                        float wgt = dec.alpha * t_before;
                        v[0] = g0 * wgt;
                        v[1] = g1 * wgt;
                        v[2] = g2 * wgt;
                        float d_alpha = g0 * fmaf(s2.x, t_before, -b0 * rc) +
                                        g1 * fmaf(s2.y, t_before, -b1 * rc) +
                                        g2 * fmaf(s2.z, t_before, -b2 * rc);
                        if (dec.gate) {
                            v[3] = d_alpha * dec.w;
                            float d_m = d_alpha * s1.y * dec.dwdm;
                            v[4] = d_m * dx * dx;
                            v[5] = d_m * dx * dy;
                            v[6] = d_m * dy * dy;
                            v[7] = -d_m * fmaf(2.f * s0.z, dx, s0.w * dy);
                            e = -d_m * fmaf(s0.w, dx, 2.f * s1.x * dy);
                        }
                        b0 = fmaf(s2.x, wgt, b0);
                        b1 = fmaf(s2.y, wgt, b1);
                        b2 = fmaf(s2.z, wgt, b2);
                        T = t_before;
                    }
                }
                if (__any_sync(kFull, hit)) {
                    float s = warp_reduce9(v, e, lane);
                    float* dst = grads + (size_t)idx * DARBS_GRADS_PER_SPLAT;
                    if (owner) atomicAdd(dst + vi, s * vmul);
                    if (lane == 1) atomicAdd(dst + 8, e);
                }
            }
            __syncwarp();
        }
        cur = nxt;
    }
    nexact = __reduce_add_sync(kFull, nexact);
    if (lane == 0 && nexact) atomicAdd(counters + CNT_EXACT, (unsigned long long)nexact);
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

darbs_status launch_render_fwd(darbs_cuda_ctx* ctx, const KParams& kp, int width, int height,
                               const float bg[3], float* image, float* t_final,
                               int32_t* processed, int32_t* contributors) {
    int tiles = ctx->tiles_x * ctx->tiles_y;
    if (tiles == 0) return DARBS_OK;
    auto* counters = (unsigned long long*)ctx->counters.ptr;
    const float4* recs = (const float4*)ctx->recs.ptr;
    const int2* ranges = (const int2*)ctx->ranges.ptr;
    const int* plist = point_list_ptr(ctx);
#define DARBS_LAUNCH_FWD(F)                                                                     \
    render_fwd_kernel<F><<<tiles, kThreads, 0, ctx->stream>>>(                                  \
        kp, recs, ranges, plist, width, height, ctx->tiles_x, bg[0], bg[1], bg[2], image,       \
        t_final, processed, contributors, counters)
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

darbs_status launch_render_bwd(darbs_cuda_ctx* ctx, const KParams& kp, int width, int height,
                               const float bg[3], const float* grad_image, const float* t_final,
                               const int32_t* processed, int64_t n, float* grads) {
    DARBS_CUDA_TRY(ctx, cudaMemsetAsync(grads, 0, sizeof(float) * DARBS_GRADS_PER_SPLAT * (size_t)n,
                                        ctx->stream));
    int tiles = ctx->tiles_x * ctx->tiles_y;
    if (tiles == 0 || n == 0) return DARBS_OK;
    auto* counters = (unsigned long long*)ctx->counters.ptr;
    const float4* recs = (const float4*)ctx->recs.ptr;
    const int2* ranges = (const int2*)ctx->ranges.ptr;
    const int* plist = point_list_ptr(ctx);
#define DARBS_LAUNCH_BWD(F)                                                                    \
    render_bwd_kernel<F><<<tiles, kThreads, 0, ctx->stream>>>(                                 \
        kp, recs, ranges, plist, width, height, ctx->tiles_x, bg[0], bg[1], bg[2], grad_image, \
        t_final, processed, grads, counters)
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
