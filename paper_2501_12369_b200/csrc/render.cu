// render.cu — block culling, per-tile front-to-back compositing (forward) and its
// reverse traversal (backward) for the DARBF families, hand-written for sm_100a.
//
// Reference semantics: darbs::forward  src/rasterizer.cpp:55-112 (inner loop :85-107)
//                      darbs::backward src/rasterizer.cpp:147-234 (inner loop :175-214)
//
// Design.  A 16x16 tile (the reference's kTileSize, so bins are
// comparable entry for entry) is split into eight 8x4 pixel blocks, one warp each.
//
//   cull_kernel   one CTA per tile walks the tile's depth-sorted list once and tests
//                 every entry against the eight blocks (exact minimum of the conic's
//                 quadratic form over the block against the splat's decision
//                 threshold).  Survivors are written, in list order, to one compact
//                 stream per block as ready-to-composite 48-byte entries
//                 { mu.x, mu.y, A, C } { B, opacity, thr_m, list position }
//                 { r, g, b, splat index }.
//   render_fwd    a warp streams its block's entries into shared memory with 1-D
//                 bulk async copies (cp.async.bulk + mbarrier: UBLKCP in SASS), three
//                 chunks of 32 entries deep, and composites them front to back in
//                 branch-free groups of eight.  No CTA-wide barrier: a warp whose 32
//                 pixels have saturated leaves immediately.
//   render_bwd    the same stream walked from the back, two sweeps per batch of 16
//                 entries (see below), 128-bit atomics into the per-splat gradients.
//
// Entries culled at block level are still COUNTED (processed[] is positional), so the
// per-pixel aux is identical to the reference's.
//
// Threshold decisions (alpha >= 1/255, dm2 vs cutoff, dm2 < 0) are taken in FP32
// against a per-splat precomputed boundary; when the FP32 value lies inside a guard
// band of that boundary the decision is re-taken in FP64 with the reference's own
// expression order, so integer outputs match the FP64 reference.
#include "splat.cuh"

namespace darbs_b200 {

namespace {

constexpr int kBlocksPerTile = 8;  // 2 x 4 blocks of 8 x 4 pixels
constexpr int kWarpsPerCta = 4;  // cull CTA: one tile, 128 list entries per step
constexpr int kThreads = 32 * kWarpsPerCta;
constexpr unsigned kFull = 0xffffffffu;

// counters (u64 each): 3 = surviving (block, entry) pairs, 4 = FP64 re-decisions,
// 5 = pixels whose transmittance came within the guard band of the floor.
// 6 = (block, entry) pairs the forward composited (before its early exits cut the streams short).
enum { CNT_SURVIVORS = 3, CNT_EXACT = 4, CNT_TFLOOR = 5, CNT_COMPOSITED = 6 };

// ------------------------------------------------------------------ packing
__global__ void pack_kernel(KParams kp, int64_t n, const float* __restrict__ mu2,
                            const float* __restrict__ conic, const float* __restrict__ opacity,
                            const float* __restrict__ rgb, float4* __restrict__ recs) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    splat_record(kp, mu2[2 * i], mu2[2 * i + 1], conic[3 * i], conic[3 * i + 1], conic[3 * i + 2], opacity[i],
                 rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2], recs + kRecVecs * i);
}

// ------------------------------------------------------------ shared pieces

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
struct ExactVisit {
    double alpha, w, dw;  // clamped alpha, weight, d weight / d dm2
    bool hit, unclamped;
};
__device__ __forceinline__ ExactVisit exact_visit(const KParams& kp, const float4* __restrict__ recs, int idx,
                                                  float fx, float fy) {
    const float4 v0 = __ldg(recs + kRecVecs * (int64_t)idx);
    const float4 v1 = __ldg(recs + kRecVecs * (int64_t)idx + 1);
    const float4 v3 = __ldg(recs + kRecVecs * (int64_t)idx + 3);
    double dx = (double)fx - (double)v0.x, dy = (double)fy - (double)v0.y;
    double a = v3.x, b = v3.y, c = v3.z, o = v1.y;
    double dm2 = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(a, dx), dx),
                                     __dmul_rn(__dmul_rn(__dmul_rn(2.0, b), dx), dy)),
                           __dmul_rn(__dmul_rn(c, dy), dy));
    ExactVisit v;
    v.alpha = v.w = v.dw = 0.0;
    v.hit = v.unclamped = false;
    if (!(dm2 >= 0.0)) return v;  // dm2 < 0 (or NaN, which the reference rejects)
    eval_exact(kp, dm2, v.w, v.dw);
    const double alpha_raw = o * v.w;
    const double alpha = fmin(kAlphaClampD, alpha_raw);
    if (alpha < kAlphaSkipD) return v;
    v.alpha = alpha;
    v.hit = true;
    v.unclamped = alpha_raw < kAlphaClampD;
    return v;
}

__device__ __noinline__ float4 exact_decide(const KParams& kp, const float4* __restrict__ recs,
                                            int idx, float fx, float fy) {
    const ExactVisit v = exact_visit(kp, recs, idx, fx, fy);
    float4 out = make_float4(0.f, 0.f, 0.f, __int_as_float(0));
    if (!v.hit) return out;
    out.x = (float)v.alpha;
    out.y = (float)v.w;
    out.z = (float)(v.dw / (double)kp.scale);
    out.w = __int_as_float(1 | (v.unclamped ? 2 : 0));
    return out;
}

// One pixel composited in FP64 as the reference does it (rasterizer.cpp:85-107), by the whole
// warp: lane j evaluates entry base + j of the block's stream, a warp scan gives every entry the
// transmittance in front of it, and the first entry that takes it below the floor ends the walk.
// Called for the few pixels per thousand whose FP32 transmittance came within the guard band of
// the floor, where the FP32 value cannot say which entry was the last (rasterizer.cpp:100).  The
// factors (1 - alpha) are the reference's; only the association of their product differs (the
// scan), a relative 1e-15 against a guard band of 1e-5.  Entries culled at block level cannot
// contribute, so the stream holds every entry that matters.
struct ExactPixel {
    double T, c0, c1, c2;
    int processed, contributors, stream_end;  // stream_end: entries of the stream the pixel consumed
};
__device__ __noinline__ ExactPixel exact_pixel(const KParams& kp, const float4* __restrict__ recs,
                                               const float4* __restrict__ stream, int n, int list_len,
                                               float fx, float fy, int lane) {
    constexpr unsigned kAll = 0xffffffffu;
    ExactPixel r;
    r.T = 1.0;
    r.contributors = 0;
    r.processed = list_len;
    r.stream_end = n;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;  // this lane's share of the colour
    for (int base = 0; base < n; base += 32) {
        const int e = base + lane;
        ExactVisit v;
        v.alpha = 0.0;
        v.hit = false;
        float4 s2 = make_float4(0.f, 0.f, 0.f, 0.f);
        int pos = 0;
        if (e < n) {
            s2 = __ldg(stream + (size_t)e * 3 + 2);
            pos = __float_as_int(__ldg(stream + (size_t)e * 3 + 1).w);
            if (__float_as_int(s2.w) >= 0) v = exact_visit(kp, recs, __float_as_int(s2.w), fx, fy);
        }
        double P = 1.0 - v.alpha;  // inclusive prefix product of the factors (alpha = 0: no hit)
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const double t = __shfl_up_sync(kAll, P, d);
            if (lane >= d) P *= t;
        }
        double before = __shfl_up_sync(kAll, P, 1);
        before = r.T * (lane == 0 ? 1.0 : before);
        const double after = r.T * P;
        const unsigned hits = __ballot_sync(kAll, v.hit);
        const unsigned cross = __ballot_sync(kAll, v.hit && after < 1e-4);  // kTransmittanceFloor
        const int jc = cross ? __ffs(cross) - 1 : 31;
        if (v.hit && lane <= jc) {
            const double at = v.alpha * before;
            a0 += (double)s2.x * at;
            a1 += (double)s2.y * at;
            a2 += (double)s2.z * at;
        }
        r.contributors += __popc(hits & (0xffffffffu >> (31 - jc)));
        r.T = __shfl_sync(kAll, after, jc);
        if (cross) {
            r.processed = __shfl_sync(kAll, pos, jc) + 1;
            r.stream_end = base + jc + 1;
            break;
        }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        a0 += __shfl_xor_sync(kAll, a0, d);
        a1 += __shfl_xor_sync(kAll, a1, d);
        a2 += __shfl_xor_sync(kAll, a2, d);
    }
    r.c0 = a0;
    r.c1 = a1;
    r.c2 = a2;
    return r;
}

// FP32 decision of one (pixel, entry) visit.  m = scaled squared Mahalanobis
// distance, computed by the caller with a fixed FMA order shared by forward
// and backward so that both passes take identical decisions.  `near` flags a
// value inside the guard band of a threshold (re-decided in FP64 when
// kp.exact); a_raw = opacity * weight, unclamped.  CLAMPBAND: also watch the band of the alpha
// clamp (the backward's gate, rasterizer.cpp:202).
template <int FAM, bool GRAD, bool CLAMPBAND = GRAD>
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
        if (CLAMPBAND) near = near || !(fabsf(a_raw - kAlphaClampF) > 2e-6f);
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
        if (CLAMPBAND) near = near || !(fabsf(a_raw - kAlphaClampF) > 2e-6f);
    }
}

// m = A dx^2 + B dx dy + C dy^2 for a record / stream entry { mu.x, mu.y, A, C } { B, ... }: the
// pairs (A, C) and (dx, dy) meet in one packed multiply, four instructions in all.  d = mu - centre
// (the form is even).  Forward and backward share this exact sequence, so both passes see the
// same bits and take identical decisions.
__device__ __forceinline__ float quad_m(const float4& e0, float B, float2 neg_centre) {
    const float2 d = __fadd2_rn(make_float2(e0.x, e0.y), neg_centre);
    const float2 pq = __fmul2_rn(make_float2(e0.z, e0.w), d);  // (A dx, C dy)
    return fmaf(fmaf(B, d.x, pq.y), d.y, pq.x * d.x);
}


// ------------------------------------------------------------ survivor streams
// One stream entry = three float4 (48 B).  A chunk = 32 entries = 1536 B, the unit
// of the bulk copies.  Streams are padded with null entries (zero opacity, threshold
// -inf, position past every list, splat index -1: nothing can take them) up to a
// multiple of kPad entries, the coarsest unit a compositing loop touches (the forward
// works in groups of 8, the backward in batches of 16), so no loop ever sees a partial
// group.  The bulk copies still move whole chunks; what lies between the padding and the
// end of the chunk is never interpreted.
constexpr int kEntryVecs = 3;
constexpr int kChunk = 32;
constexpr int kPad = 16;
constexpr int kChunkVecs = kChunk * kEntryVecs;
constexpr int kChunkBytes = kChunkVecs * (int)sizeof(float4);

// Entry offset of block `blk`'s stream for tile `tile` whose point list is [beg, end):
// every block owns a region as long as the tile's list rounded up to a chunk (the
// worst case).  8 (K + 32 tiles) entries of address space; only survivors and their
// padding are ever written or read.
__host__ __device__ __forceinline__ size_t stream_offset(int tile, int beg, int end, int blk) {
    const size_t cap = (size_t)((end - beg + kChunk - 1) & ~(kChunk - 1));
    return (size_t)kBlocksPerTile * ((size_t)beg + (size_t)kChunk * (size_t)tile) + (size_t)blk * cap;
}

__device__ __forceinline__ void store_null_entry(float4* e) {
    e[0] = make_float4(0.f, 0.f, 0.f, 0.f);
    e[1] = make_float4(0.f, 0.f, -3.0e38f, __int_as_float(0x7fffffff));
    e[2] = make_float4(0.f, 0.f, 0.f, __int_as_float(-1));
}

// ------------------------------------------------------------------ culling
// Lower bound of m(d) = A dx^2 + B dx dy + C dy^2 over the rectangle of pixel
// centres [X0,X1]x[Y0,Y1] (d measured from the splat centre), for A, C > 0 and
// 4AC > B^2 (the pack kernel sends every other conic down the NaN path).  The
// minimum of a convex quadratic over a box that does not contain the unconstrained
// minimiser lies on an edge facing it; evaluated branch-free: candidate 1 = best
// point of the vertical line through the x-clamped centre, candidate 2 = same for
// the horizontal line; when the centre is inside the box both are 0, when it is
// outside along one axis only the candidate of the other axis lies on the facing
// edge too and is not smaller.  (dxc, ex0, ex1) / (dyc, ey0, ey1): clamped centre
// and box edges per axis, shared between the blocks of a row / column.
__device__ __forceinline__ bool block_survives(float A, float B, float C, float kx, float ky,
                                               float thr2, float dxc, float ex0, float ex1,
                                               float dyc, float ey0, float ey1) {
    const float dy1 = fminf(fmaxf(kx * dxc, ey0), ey1);
    const float m1 = fmaf(fmaf(A, dxc, B * dy1), dxc, (C * dy1) * dy1);
    const float dx2 = fminf(fmaxf(ky * dyc, ex0), ex1);
    const float m2 = fmaf(fmaf(A, dx2, B * dyc), dx2, (C * dyc) * dyc);
    // Per-pixel decisions can only be positive for m <= thr + band; keep a relative
    // margin for the FP32 rounding of the bound itself.  A NaN threshold (decided in
    // FP64) compares false and survives.
    return !(fminf(m1, m2) * 0.9999f > thr2);
}

// One CTA per tile; thread t of a 256-entry step takes list entry base + t, gathers its
// record and tests it against the eight blocks.  Per block, a ballot per warp and a
// prefix over the eight warps give every survivor its slot, so streams keep list order.
__global__ void __launch_bounds__(kThreads)
cull_kernel(KParams kp, const float4* __restrict__ recs, const int2* __restrict__ ranges,
            const int* __restrict__ point_list, int tiles_x, int seg, float4* __restrict__ streams,
            int* __restrict__ stream_count, unsigned long long* __restrict__ counters,
            const int* __restrict__ tile_order) {
    __shared__ int wcnt[kWarpsPerCta][kBlocksPerTile];
    __shared__ int wpre[kWarpsPerCta][kBlocksPerTile];
    // CTAs take the tiles longest list first (binning.cu tile_order_kernel); raster order without it
    const int tile = tile_order ? tile_order[blockIdx.x] : blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int2 range = ranges[tile];
    const int beg = range.x, list_end = range.y;
    // only the first `seg` entries of the list are culled here: the forward extends a block's stream
    // itself when its pixels outlive them (extend_stream), and most blocks of a dense scene do not
    const int end = list_end - beg > seg ? beg + seg : list_end;
    const float tx0 = (float)((tile % tiles_x) * DARBS_TILE_SIZE) + 0.5f;
    const float ty0 = (float)((tile / tiles_x) * DARBS_TILE_SIZE) + 0.5f;
    const float band2 = 2.f * kp.band;
    const unsigned lt_mask = (1u << lane) - 1u;
    // threads 0..63 keep the running stream length of block (tid & 7); the eight copies agree
    int run = 0;
    float4* const tile_streams = streams + kEntryVecs * stream_offset(tile, beg, list_end, 0);
    const size_t cap = (size_t)((list_end - beg + kChunk - 1) & ~(kChunk - 1));

    // software pipeline: list index two steps ahead, record one step ahead of the step under test
    int idx_n = beg + tid < end ? __ldg(point_list + beg + tid) : -1;
    float4 n0 = make_float4(0.f, 0.f, 0.f, 0.f), n1 = n0, n2 = n0;
    if (idx_n >= 0) {
        const float4* r = recs + kRecVecs * (int64_t)idx_n;
        n0 = __ldg(r);
        n1 = __ldg(r + 1);
        n2 = __ldg(r + 2);
    }
    int idx_nn = beg + kThreads + tid < end ? __ldg(point_list + beg + kThreads + tid) : -1;
    for (int base = beg; base < end; base += kThreads) {
        const int k = base + tid;
        const bool valid = k < end;
        const float4 v0 = n0, v1 = n1, v2 = n2;
        const int idx = idx_n;
        idx_n = idx_nn;
        if (idx_n >= 0) {
            const float4* r = recs + kRecVecs * (int64_t)idx_n;
            n0 = __ldg(r);
            n1 = __ldg(r + 1);
            n2 = __ldg(r + 2);
        }
        idx_nn = k + 2 * kThreads < end ? __ldg(point_list + k + 2 * kThreads) : -1;
        unsigned bits = 0;
        if (valid) {
            const float thr2 = v1.z + band2;
            float dxc[2], ex0[2], ex1[2];
#pragma unroll
            for (int xb = 0; xb < 2; ++xb) {
                ex0[xb] = tx0 + 8.f * xb - v0.x;
                ex1[xb] = ex0[xb] + 7.f;
                dxc[xb] = fminf(fmaxf(0.f, ex0[xb]), ex1[xb]);
            }
#pragma unroll
            for (int yb = 0; yb < 4; ++yb) {
                const float ey0 = ty0 + 4.f * yb - v0.y, ey1 = ey0 + 3.f;
                const float dyc = fminf(fmaxf(0.f, ey0), ey1);
#pragma unroll
                for (int xb = 0; xb < 2; ++xb)
                    if (block_survives(v0.z, v1.x, v0.w, v1.w, v2.w, thr2, dxc[xb], ex0[xb], ex1[xb], dyc, ey0,
                                       ey1))
                        bits |= 1u << (yb * 2 + xb);
            }
        }
        unsigned masks[kBlocksPerTile];
#pragma unroll
        for (int b = 0; b < kBlocksPerTile; ++b) masks[b] = __ballot_sync(kFull, (bits >> b) & 1u);
        if (lane < kBlocksPerTile) {
            unsigned m = masks[0];
#pragma unroll
            for (int b = 1; b < kBlocksPerTile; ++b) m = lane == b ? masks[b] : m;
            wcnt[warp][lane] = __popc(m);
        }
        __syncthreads();
        if (tid < kWarpsPerCta * kBlocksPerTile) {
            const int w = tid >> 3, b = tid & 7;
            int pre = run, total = 0;
#pragma unroll
            for (int ww = 0; ww < kWarpsPerCta; ++ww) {
                const int c = wcnt[ww][b];
                pre += ww < w ? c : 0;
                total += c;
            }
            wpre[w][b] = pre;
            run += total;
        }
        __syncthreads();
        if (bits) {
            const float4 e1 = make_float4(v1.x, v1.y, v1.z, __int_as_float(k - beg));
            const float4 e2 = make_float4(v2.x, v2.y, v2.z, __int_as_float(idx));
#pragma unroll
            for (int b = 0; b < kBlocksPerTile; ++b)
                if ((bits >> b) & 1u) {
                    const size_t slot = (size_t)b * cap + (size_t)(wpre[warp][b] + __popc(masks[b] & lt_mask));
                    float4* e = tile_streams + kEntryVecs * slot;
                    e[0] = v0;
                    e[1] = e1;
                    e[2] = e2;
                }
        }
        // wcnt / wpre are rewritten only after the next step's first barrier / by the threads
        // that passed this step's second barrier, so no third barrier is needed
    }
    // stream lengths, and null padding up to a whole chunk
    __shared__ int total[kBlocksPerTile];
    if (tid < kBlocksPerTile) {
        total[tid] = run;
        stream_count[tile * kBlocksPerTile + tid] = run;
        atomicAdd(counters + CNT_SURVIVORS, (unsigned long long)run);
    }
    __syncthreads();
    for (int b = warp; b < kBlocksPerTile; b += kWarpsPerCta) {
        const int n = total[b];
        const int padded = (n + kPad - 1) & ~(kPad - 1);
        if (n + lane < padded) store_null_entry(tile_streams + kEntryVecs * ((size_t)b * cap + (size_t)(n + lane)));
    }
}

// ---------------------------------------------------- bulk async copies (TMA)
__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// One lane arms the barrier with the byte count and issues the copy, which arrives on it.
__device__ __forceinline__ void bulk_load(float4* dst, const float4* src, unsigned bytes,
                                          unsigned long long* bar) {
    const unsigned b = smem_addr(bar);
    // earlier generic-proxy reads of dst (previous use of the stage) are ordered before the
    // async-proxy write by the __syncwarp that precedes this call plus this proxy fence
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(b)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_LOOP:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@p bra WAIT_DONE;\n"
        "bra WAIT_LOOP;\n"
        "WAIT_DONE:\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

// ------------------------------------------------------------------ forward
// Entries composited speculatively between two guard-band checks, and the granularity at which a
// warp whose pixels have saturated leaves.  Measured per family: the Gaussian, most of whose
// blocks run their whole stream, prefers 16 (half the per-group bookkeeping: -1 %); the families
// whose pixels saturate early prefer 8 (fewer dead visits before the exit: -1 to -2 %).
constexpr int kGroupMax = 16;
// Stages of the forward's bulk-copy ring.  A block that saturates early leaves with the copies in
// flight still to land and their bytes read for nothing: one chunk of prefetch distance for those
// families, two for the Gaussian.
template <int FAM>
struct FwdStages {
    static constexpr int value = FAM == FAM_GAUSS2 ? 3 : 2;
};
template <int FAM>
struct FwdGroup {
    static constexpr int value = FAM == FAM_GAUSS2 ? 16 : 8;
};

// A pixel is live while its transmittance is at or above the floor
// (rasterizer.cpp:100 leaves the loop the first time T < 1e-4); lanes outside
// the image start at T = 0 and never take a splat.
struct FwdPixel {
    float2 crg;  // red and green accumulate in one packed FMA
    float T, cb;
    float contrib;  // contributor count, kept in FP32 (exact below 2^24) so a hit costs one FADD
    int nlive;      // stream entries met while live: the last of them is the one that crossed the floor
    unsigned nexact;
};

// Opacity from which alpha = o * w can reach the 0.99 clamp (rasterizer.cpp:93); FP32 weights
// exceed 1 by rounding only.  Groups without such an entry run a variant without the clamp.
constexpr float kClampableF = 0.98f;

// Front-to-back compositing of one queued survivor into this lane's pixel
// (rasterizer.cpp:88-100).  Branch-free: a lane that does not take the splat
// blends alpha = 0.
//
// CAREFUL = false is the speculative form the batch loop runs over a group of
// survivors: it only records in near_acc whether any FP32 value fell inside
// the guard band of a threshold; the group is then replayed from the saved
// pixel state with CAREFUL = true, which re-takes those decisions in FP64.
template <int FAM, bool CAREFUL, bool CLAMP>
__device__ __forceinline__ void fwd_visit(const KParams& kp, const float4* __restrict__ recs,
                                          const float4* __restrict__ qe, float fx, float fy,
                                          FwdPixel& px, bool& near_acc) {
    const float4 s0 = qe[0];
    const float4 s1 = qe[1];
    const float4 s2 = qe[2];
    const float m = quad_m(s0, s1.x, make_float2(-fx, -fy));
    if constexpr (!CAREFUL && FAM != FAM_GENERIC) {
        // The speculative form, two instructions shorter than what the compiler makes of the
        // general one below: take = (thr > m) && live selects alpha, and both counters (visits met
        // while live, contributors) are predicated adds.  live = !(T < floor), as below.
        near_acc = near_acc || !(fabsf(s1.z - m) > kp.band);  // also true for a NaN threshold
        const float a_raw = s1.y * fam_weight<FAM>(m);
        float alpha = CLAMP ? fminf(kAlphaClampF, a_raw) : a_raw;
        asm("{\n\t"
            ".reg .pred p, q;\n\t"
            "setp.geu.f32 p, %5, %6;\n\t"
            "setp.gt.and.f32 q, %3, %4, p;\n\t"
            "@p add.s32 %1, %1, 1;\n\t"
            "@q add.f32 %2, %2, 0f3F800000;\n\t"
            "selp.f32 %0, %0, 0f00000000, q;\n\t"
            "}"
            : "+f"(alpha), "+r"(px.nlive), "+f"(px.contrib)
            : "f"(s1.z), "f"(m), "f"(px.T), "f"(kTFloorF));
        const float at = alpha * px.T;
        px.crg = __ffma2_rn(make_float2(s2.x, s2.y), make_float2(at, at), px.crg);
        px.cb = fmaf(s2.z, at, px.cb);
        px.T = fmaf(-alpha, px.T, px.T);
        return;
    }
    const bool live = !(px.T < kTFloorF);
    bool hit, near;
    float a_raw, w, dwdm;
    fast_decide<FAM, false>(kp, m, s1.z, s1.y, hit, near, a_raw, w, dwdm);
    float alpha = CLAMP ? fminf(kAlphaClampF, a_raw) : a_raw;
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
    const bool take = hit && live;
    alpha = take ? alpha : 0.f;
    // rasterizer.cpp:96-100
    const float at = alpha * px.T;
    px.crg = __ffma2_rn(make_float2(s2.x, s2.y), make_float2(at, at), px.crg);
    px.cb = fmaf(s2.z, at, px.cb);
    px.contrib += take ? 1.f : 0.f;
    // T never rises and a dead lane blends alpha = 0, so the entries a lane meets while live are a
    // prefix of the stream and the last of them is the one that crossed the floor
    if (live) ++px.nlive;
    px.T = fmaf(-alpha, px.T, px.T);
}

// The cull kernel covers only the first `seg` entries of a tile's list.  A block whose pixels are
// still live at the end of its stream culls on by itself: the warp tests the next list entries
// (lane = entry) against its own 8x4 block with the cull kernel's bound and appends the survivors
// at position n of its stream, in list order, until a chunk's worth has been added or the list
// ends; null padding follows up to a multiple of kPad, as behind every stream.  Returns the new
// stream length.  Only this warp reads the new entries before the kernel ends (plain loads).
__device__ __noinline__ int extend_stream(const KParams& kp, const float4* __restrict__ recs,
                                          const int* __restrict__ list, int list_len, int& culled,
                                          float4* __restrict__ dst, int n, float bx05, float by05, int lane) {
    // (`culled` by reference: the callers are slow paths that hold it in a local of their own)
    const float band2 = 2.f * kp.band;
    const unsigned lt = (1u << lane) - 1u;
    int count = 0;
    while (culled < list_len && count < kChunk) {
        const int k = culled + lane;
        bool surv = false;
        float4 v0 = make_float4(0.f, 0.f, 0.f, 0.f), v1 = v0, v2 = v0;
        int idx = -1;
        if (k < list_len) {
            idx = __ldg(list + k);
            const float4* r = recs + kRecVecs * (int64_t)idx;
            v0 = __ldg(r);
            v1 = __ldg(r + 1);
            v2 = __ldg(r + 2);
            const float ex0 = bx05 - v0.x, ex1 = ex0 + 7.f, dxc = fminf(fmaxf(0.f, ex0), ex1);
            const float ey0 = by05 - v0.y, ey1 = ey0 + 3.f, dyc = fminf(fmaxf(0.f, ey0), ey1);
            surv = block_survives(v0.z, v1.x, v0.w, v1.w, v2.w, v1.z + band2, dxc, ex0, ex1, dyc, ey0, ey1);
        }
        const unsigned m = __ballot_sync(kFull, surv);
        if (surv) {
            float4* e = dst + kEntryVecs * (size_t)(n + count + __popc(m & lt));
            e[0] = v0;
            e[1] = make_float4(v1.x, v1.y, v1.z, __int_as_float(k));
            e[2] = make_float4(v2.x, v2.y, v2.z, __int_as_float(idx));
        }
        count += __popc(m);
        culled = culled + 32 < list_len ? culled + 32 : list_len;
    }
    const int n_new = n + count;
    const int padded = (n_new + kPad - 1) & ~(kPad - 1);
    if (n_new + lane < padded) store_null_entry(dst + kEntryVecs * (size_t)(n_new + lane));
    __threadfence();
    __syncwarp();
    return n_new;
}

// The slow path of the forward for a block that outlives the culled part of its list: composite
// what the stream holds (whole groups; straight from global memory, no ring), extend the stream by
// about a chunk, and so on until the pixels saturate or the list ends.  `pos` is the first stream
// entry not yet composited; it comes back as the forward's `used`.  Always the clamp-aware visit.
struct TailResult {  // by value in and out: nothing of the kernel's loop state has its address taken
    FwdPixel px;
    int pos, n, culled;
};
template <int FAM>
__device__ __noinline__ TailResult forward_tail(const KParams& kp, const float4* __restrict__ recs,
                                                const int* __restrict__ list, int list_len, int culled,
                                                float4* __restrict__ dst, int n, int pos, float bx05, float by05,
                                                float fx, float fy, int lane, FwdPixel px, float4* __restrict__ smem,
                                                int smem_entries) {
    constexpr int kGroup = FwdGroup<FAM>::value;
    bool dead = false;
    while (true) {
        const bool last_round = culled >= list_len;
        const int n_run = last_round ? n : n - n % kGroup;  // the last group may run into the null padding
        while (pos < n_run && !dead) {
            // the warp's ring is idle here: the next entries are staged in it by plain copies (the warp
            // wrote them itself a moment ago), so a visit reads shared memory as in the stream walk
            const int batch = min(((n_run - pos + kGroup - 1) / kGroup) * kGroup, smem_entries);
            __syncwarp();
            for (int i = lane; i < batch * kEntryVecs; i += 32) smem[i] = dst[(size_t)pos * kEntryVecs + i];
            __syncwarp();
            for (int b = 0; b < batch && !dead; b += kGroup, pos += kGroup) {
                const float4* qb = smem + b * kEntryVecs;
                const FwdPixel save = px;
                bool near_acc = false;
                for (int j = 0; j < kGroup; ++j) fwd_visit<FAM, false, true>(kp, recs, qb + j * 3, fx, fy, px, near_acc);
                if (kp.exact && __any_sync(kFull, near_acc)) {
                    px = save;
                    for (int j = 0; j < kGroup; ++j) fwd_visit<FAM, true, true>(kp, recs, qb + j * 3, fx, fy, px, near_acc);
                }
                dead = !__any_sync(kFull, !(px.T < kTFloorF));
            }
        }
        if (dead || last_round) break;
        n = extend_stream(kp, recs, list, list_len, culled, dst, n, bx05, by05, lane);
    }
    TailResult r;
    r.px = px;
    r.pos = pos;
    r.n = n;
    r.culled = culled;
    return r;
}

// Warps of a forward CTA.  A warp owns one 8x4 block and leaves as soon as its 32 pixels have
// saturated; with a whole tile (8 warps) per CTA the early leavers' slots idle until the CTA's
// slowest warp is done, so CTAs are kept small and the hardware scheduler backfills.
constexpr int kFwdWarps = 2;

// TAIL: the cull kernel covered only the first `seg` entries of the lists, so a block may have to
// cull on by itself (forward_tail).  Without it the kernel is the plain stream walk.
template <int FAM, bool TAIL>
__global__ void __launch_bounds__(32 * kFwdWarps, 32 / kFwdWarps)
render_fwd_kernel(KParams kp, const float4* __restrict__ recs, const int2* __restrict__ ranges,
                  const int* __restrict__ point_list, int seg, const float4* __restrict__ streams,
                  const int* __restrict__ stream_count, int* __restrict__ stream_used, int W, int H,
                  int tiles_x, float bg0, float bg1, float bg2, float* __restrict__ image,
                  float* __restrict__ t_final, int* __restrict__ processed, int* __restrict__ contributors,
                  unsigned long long* __restrict__ counters, const int* __restrict__ tile_order) {
    constexpr int kGroup = FwdGroup<FAM>::value;
    constexpr int kDepth = FwdStages<FAM>::value;  // stages of the bulk-copy ring
    __shared__ __align__(128) float4 ring[kFwdWarps][kDepth][kChunkVecs];
    __shared__ unsigned long long bars[kFwdWarps][kDepth];
    // the warp index through a warp reduction: the compiler then knows it is warp-uniform and
    // keeps the ring pointers and loop control in uniform registers
    const int lwarp = __reduce_min_sync(kFull, (int)(threadIdx.x >> 5)), lane = threadIdx.x & 31;
    const int gwarp = blockIdx.x * kFwdWarps + lwarp;
    const int warp = gwarp % kBlocksPerTile;  // the block inside the tile
    const int tile = tile_order ? tile_order[gwarp / kBlocksPerTile] : gwarp / kBlocksPerTile;
    const int bx = (tile % tiles_x) * DARBS_TILE_SIZE + (warp & 1) * 8;
    const int by = (tile / tiles_x) * DARBS_TILE_SIZE + (warp >> 1) * 4;
    if (bx >= W || by >= H) return;  // whole block outside the image
    const int pxl = bx + (lane & 7), pyl = by + (lane >> 3);
    const bool inside = pxl < W && pyl < H;
    const float fx = pxl + 0.5f, fy = pyl + 0.5f;
    const int2 range = ranges[tile];
    const int beg = range.x, end = range.y;

    FwdPixel px;
    px.T = inside ? 1.f : 0.f;
    px.crg = make_float2(0.f, 0.f);
    px.cb = 0.f;
    px.contrib = 0.f;
    px.nlive = 0;
    px.nexact = 0;

    const float4* src = streams + kEntryVecs * stream_offset(tile, beg, end, warp);
    const int n_culled = stream_count[tile * kBlocksPerTile + warp];
    // While the stream can still grow (the cull kernel covered only the first `seg` entries of the
    // list) only whole groups are composited here: the entries past the last whole group wait for
    // forward_tail, which appends right behind them (there is no padding inside a stream).
    const int n = (TAIL && end - beg > seg) ? n_culled - n_culled % kGroup : n_culled;
    const int nchunks = (n + kChunk - 1) / kChunk;
    float4* stage0 = ring[lwarp][0];
    unsigned long long* bar = bars[lwarp];
    if (lane == 0) {
        for (int s = 0; s < kDepth; ++s) mbar_init(bar + s);
        mbar_init_fence();
        // chunks 0 .. kDepth - 2 in flight before the loop; chunk c + kDepth - 1 is issued while c is composited
        for (int s = 0; s < kDepth - 1; ++s)
            if (nchunks > s) bulk_load(stage0 + s * kChunkVecs, src + (size_t)s * kChunkVecs, kChunkBytes, bar + s);
    }
    __syncwarp();
    int used = 0, stage = 0;
    unsigned parity = 0;
    int c = 0;
    for (; c < nchunks; ++c) {
        if (lane == 0 && c + kDepth - 1 < nchunks) {
            const int fill = stage == 0 ? kDepth - 1 : stage - 1;  // the stage chunk c - 1 vacated
            bulk_load(stage0 + fill * kChunkVecs, src + (size_t)(c + kDepth - 1) * kChunkVecs, kChunkBytes, bar + fill);
        }
        mbar_wait(bar + stage, parity);
        const float4* qc = stage0 + stage * kChunkVecs;
        const int rem = n - c * kChunk;
        const int ngroups = rem >= kChunk ? kChunk / kGroup : (rem + kGroup - 1) / kGroup;
        // entry `lane` of the chunk: can its alpha reach the clamp?  (What lies beyond the padding
        // is never composited; its bits only cover groups that do not run.)
        const unsigned clampable =
            FAM == FAM_GENERIC ? kFull : __ballot_sync(kFull, !(qc[lane * kEntryVecs + 1].y < kClampableF));
        // the warp leaves after the first group that finds its 32 pixels saturated (a chunk later
        // would be half a chunk of dead visits on average, a quarter of an early-terminating block)
        int g = 0;
        bool dead = false;
        for (; g < ngroups && !dead; ++g) {
            const float4* qb = qc + g * (kGroup * kEntryVecs);
            const FwdPixel save = px;
            bool near_acc = false;
            if ((clampable >> (g * kGroup)) & ((1u << kGroup) - 1u)) {
#pragma unroll
                for (int j = 0; j < kGroup; ++j)
                    fwd_visit<FAM, false, true>(kp, recs, qb + j * 3, fx, fy, px, near_acc);
            } else {
#pragma unroll
                for (int j = 0; j < kGroup; ++j)
                    fwd_visit<FAM, false, false>(kp, recs, qb + j * 3, fx, fy, px, near_acc);
            }
            if (kp.exact && __any_sync(kFull, near_acc)) {  // a few groups per thousand
                px = save;
                for (int j = 0; j < kGroup; ++j)
                    fwd_visit<FAM, true, true>(kp, recs, qb + j * 3, fx, fy, px, near_acc);
            }
            dead = !__any_sync(kFull, !(px.T < kTFloorF));
        }
        used = c * kChunk + g * kGroup;  // the backward walks [0, used)
        __syncwarp();
        if (stage == kDepth - 1) {
            stage = 0;
            parity ^= 1u;
        } else {
            ++stage;
        }
        if (dead) {
            ++c;
            break;
        }
    }
    // copies still in flight must land before the CTA's shared memory can be given away
    for (int d = c; d < nchunks && d < c + kDepth - 1; ++d) {
        mbar_wait(bar + stage, parity);
        if (stage == kDepth - 1) {
            stage = 0;
            parity ^= 1u;
        } else {
            ++stage;
        }
    }
    // Live pixels at the end of the stream and more of the list behind it: the block culls on by itself.
    int n_stream = n_culled;            // entries of the stream, for exact_pixel below
    int culled = (TAIL && end - beg > seg) ? seg : end - beg;
    if (TAIL && culled < end - beg && c >= nchunks && __any_sync(kFull, !(px.T < kTFloorF))) {
        const TailResult r = forward_tail<FAM>(kp, recs, point_list + beg, end - beg, culled, const_cast<float4*>(src),
                                               n_stream, used, (float)bx + 0.5f, (float)by + 0.5f, fx, fy, lane, px,
                                               stage0, kDepth * kChunk);
        px = r.px;
        used = r.pos;
        n_stream = r.n;
        culled = r.culled;
    }

    // Pixels whose transmittance came within the guard band of the floor: the last value (the first
    // below the floor, or the final one) and, for a pixel that crossed, the value just before the
    // crossing, recovered from the entry that crossed it.  FP32 cannot say on which entry such a
    // pixel stopped; it is composited again in FP64 by the whole warp (exact_pixel).
    bool flagged = false;
    int proc = end - beg;  // processed (rasterizer.cpp:86,100): the whole list, or up to the entry that crossed
    float out_r = fmaf(bg0, px.T, px.crg.x), out_g = fmaf(bg1, px.T, px.crg.y), out_b = fmaf(bg2, px.T, px.cb);
    float out_t = px.T;
    int out_contrib = (int)px.contrib;
    if (inside) {
        flagged = fabsf(px.T - kTFloorF) < 2e-9f;
        if (px.T < kTFloorF && px.nlive > 0) {
            const float4 v0 = __ldg(src + (size_t)(px.nlive - 1) * kEntryVecs);
            const float4 v1 = __ldg(src + (size_t)(px.nlive - 1) * kEntryVecs + 1);
            proc = __float_as_int(v1.w) + 1;
            bool hit, near;
            float a_raw, w, dwdm;
            fast_decide<FAM, false>(kp, quad_m(v0, v1.x, make_float2(-fx, -fy)), v1.z, v1.y, hit, near,
                                    a_raw, w, dwdm);
            const float t_cross = px.T / (1.0f - fminf(kAlphaClampF, a_raw));
            flagged = flagged || fabsf(t_cross - kTFloorF) < 4e-9f;
        }
    }
    unsigned todo = kp.exact ? __ballot_sync(kFull, flagged) : 0u;
    const unsigned nfloor = __popc(__ballot_sync(kFull, flagged));
    // the FP64 walk of a flagged pixel may go on past the entry its FP32 walk stopped at: it needs the
    // survivors of the whole list
    if (TAIL && todo) {
        int done = culled;  // a local of this rare path: `culled` itself keeps out of memory
        while (done < end - beg)
            n_stream = extend_stream(kp, recs, point_list + beg, end - beg, done, const_cast<float4*>(src), n_stream,
                                     (float)bx + 0.5f, (float)by + 0.5f, lane);
    }
    while (todo) {
        const int l = __ffs(todo) - 1;
        todo &= todo - 1;
        const ExactPixel ep = exact_pixel(kp, recs, src, n_stream, end - beg, __shfl_sync(kFull, fx, l),
                                          __shfl_sync(kFull, fy, l), lane);
        // the backward walks [0, used): it must reach the entry this pixel stopped on
        used = max(used, (ep.stream_end + kGroup - 1) & ~(kGroup - 1));
        if (lane == l) {
            out_r = (float)(ep.c0 + (double)bg0 * ep.T);
            out_g = (float)(ep.c1 + (double)bg1 * ep.T);
            out_b = (float)(ep.c2 + (double)bg2 * ep.T);
            out_t = (float)ep.T;
            proc = ep.processed;
            out_contrib = ep.contributors;
        }
    }
    if (inside) {
        size_t p = (size_t)pyl * W + pxl;
        image[p * 3 + 0] = out_r;
        image[p * 3 + 1] = out_g;
        image[p * 3 + 2] = out_b;
        t_final[p] = out_t;
        processed[p] = proc;
        contributors[p] = out_contrib;
    }
    // instrumentation: one atomic per warp per counter
    const unsigned nexact = __reduce_add_sync(kFull, px.nexact);
    if (lane == 0) {
        stream_used[tile * kBlocksPerTile + warp] = used;  // entries composited: all the backward needs
        atomicAdd(counters + CNT_COMPOSITED, (unsigned long long)used);
        if (n_stream > n_culled) atomicAdd(counters + CNT_SURVIVORS, (unsigned long long)(n_stream - n_culled));
        if (nexact) atomicAdd(counters + CNT_EXACT, (unsigned long long)nexact);
        if (nfloor) atomicAdd(counters + CNT_TFLOOR, (unsigned long long)nfloor);
    }
}

// ----------------------------------------------------------------- backward
//
// One single-warp CTA per 8x4 block (warps need nothing from each other, and with several
// blocks to a CTA the early finishers' slots idle until the slowest is done: measured 6-9 %
// slower at 4 warps per CTA for the families whose pixels saturate early); the warp walks the part of its stream the forward composited, from the
// back, in two sweeps per batch of kBwdBatch entries:
//   sweep 1 (lane = pixel): the reverse compositing chain of rasterizer.cpp:
//       189-213; per (pixel, entry) it leaves three numbers in a padded
//       shared-memory matrix: wgt = alpha * T_before (colour gradient weight),
//       y = d_alpha * w (opacity gradient term), z = d_alpha * o * dw/dm (the
//       common factor of the conic and mean gradients), the last two gated by
//       the alpha clamp;
//   sweep 2 (lane = entry x half of the pixels): each lane sums its entry's nine
//       gradients over 16 pixels in registers; one shuffle folds the two halves.
//       No per-entry cross-lane reduction.
// Then two 128-bit and one 32-bit red.global.add per entry into gradient rows
// padded to 12 floats.
constexpr int kBwdWarps = 1;
constexpr int kBwdThreads = 32 * kBwdWarps;
constexpr int kBwdBatch = 16;
constexpr int kBwdGroup = 8;  // sweep 1's speculative unit (16 spills at the backward's 80 registers: +12 %)
// Stages of the bulk-copy ring: one chunk (32 entries, a few thousand cycles of compositing) of
// prefetch distance hides the copy; the third stage of the forward would cost resident CTAs here.
constexpr int kBwdStages = 2;
static_assert(kPad % kBwdBatch == 0 && kPad % kGroupMax == 0 && kBwdBatch % kBwdGroup == 0 && kChunk % kPad == 0,
              "stream padding covers every loop unit");
constexpr int kXStride = kBwdBatch + 1;  // odd: conflict-free both by row and by column
constexpr int kSplatGradStride = 12;     // internal gradient rows are padded to 12 floats for 128-bit atomics

struct BwdPixel {
    float T;       // transmittance in front of the cursor
    float s;       // <g, colour composited behind the cursor> (rasterizer.cpp:180)
    float g0, g1, g2;
    int nproc;
    unsigned nexact;
};

// For the Gaussian dw/dm = -ln2 w, so z = -ln2 o y: only y is exchanged and sweep 2 scales its
// moments by -ln2 o once per entry.
template <int FAM>
struct BwdExchange {
    static constexpr bool kPair = FAM != FAM_GAUSS2;
};

template <int FAM, bool CAREFUL, bool CLAMP>
__device__ __forceinline__ void bwd_visit(const KParams& kp, const float4* __restrict__ recs,
                                          const float4* __restrict__ qe, float fx, float fy,
                                          BwdPixel& px, float* __restrict__ xw,
                                          float* __restrict__ xyz, bool& near_acc) {
    const float4 s0 = qe[0];
    const float4 s1 = qe[1];
    const float4 s2 = qe[2];
    const float m = quad_m(s0, s1.x, make_float2(-fx, -fy));
    const bool elig = __float_as_int(s1.w) < px.nproc;
    bool hit, near;
    float a_raw, w, dwdm;
    fast_decide<FAM, true, CLAMP>(kp, m, s1.z, s1.y, hit, near, a_raw, w, dwdm);
    if constexpr (!CLAMP) {
        // No entry of the group can reach the alpha clamp (opacity < kClampableF): alpha = o w, the
        // gradient always passes (rasterizer.cpp:202), and there is no clamp band to watch.
        static_assert(!CAREFUL, "the replay runs the full form");
        near_acc = near_acc || near;
        hit = hit && elig;
        float alpha;
        if constexpr (!BwdExchange<FAM>::kPair) {
            w = hit ? w : 0.f;  // zeroes alpha and the exchanged y = d_alpha w at once
            alpha = s1.y * w;
        } else {
            alpha = hit ? a_raw : 0.f;
        }
        // rasterizer.cpp:189-213 with s = <g, accum_behind>
        const float rc = rcp_approx(1.0f - alpha);
        const float t_before = px.T * rc;
        const float wgt = alpha * t_before;
        const float gc = fmaf(px.g2, s2.z, fmaf(px.g1, s2.y, px.g0 * s2.x));
        const float d_alpha = fmaf(t_before, gc, -(rc * px.s));
        *xw = wgt;
        if constexpr (BwdExchange<FAM>::kPair) {
            const float da = hit ? d_alpha : 0.f;
            *reinterpret_cast<float2*>(xyz) = make_float2(da * w, da * s1.y * dwdm);
        } else {
            *xyz = d_alpha * w;
        }
        px.s = fmaf(gc, wgt, px.s);
        px.T = t_before;  // a lane that does not take the entry: alpha = 0, rcp(1) = 1 exactly
        return;
    }
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
    if constexpr (BwdExchange<FAM>::kPair)
        *reinterpret_cast<float2*>(xyz) = make_float2(da * w, da * s1.y * dwdm);
    else
        *xyz = da * w;
    px.s = fmaf(gc, wgt, px.s);
    px.T = t_before;  // a lane that does not take the entry: alpha = 0, rcp(1) = 1 exactly
}

// fixed-point add of the deterministic mode (common.cuh kFixedScale)
__device__ __forceinline__ void fixed_add(long long* dst, float v) {
    atomicAdd(reinterpret_cast<unsigned long long*>(dst),
              (unsigned long long)__float2ll_rn(v * (float)kFixedScale));
}

// DET: the nine sums of an entry go to int64 fixed-point rows (9 per splat) instead of the padded
// float rows — order-independent, see darbs_cuda_set_deterministic.
template <int FAM, bool DET = false>
__global__ void __launch_bounds__(kBwdThreads, 24 / kBwdWarps)
render_bwd_kernel(KParams kp, const float4* __restrict__ recs, const int2* __restrict__ ranges,
                  const float4* __restrict__ streams, const int* __restrict__ stream_used, int W, int H,
                  int tiles_x, float bg0, float bg1, float bg2, const float* __restrict__ grad_image,
                  const float* __restrict__ t_final, const int* __restrict__ processed,
                  float* __restrict__ grads, unsigned long long* __restrict__ counters,
                  const int* __restrict__ tile_order) {
    __shared__ __align__(128) float4 ring[kBwdWarps][kBwdStages][kChunkVecs];
    __shared__ unsigned long long bars[kBwdWarps][kBwdStages];
    // [0]: wgt, then (y, z) pairs, or y alone for the Gaussian
    __shared__ __align__(16) float xch[kBwdWarps][BwdExchange<FAM>::kPair ? 3 : 2][32 * kXStride];
    __shared__ float4 gpix[kBwdWarps][32];
    const int warp = __reduce_min_sync(kFull, (int)(threadIdx.x >> 5)), lane = threadIdx.x & 31;
    const int gwarp = blockIdx.x * kBwdWarps + warp;
    const int blk = gwarp % kBlocksPerTile;  // the forward's block index
    const int tile = tile_order ? tile_order[gwarp / kBlocksPerTile] : gwarp / kBlocksPerTile;
    const int bx = (tile % tiles_x) * DARBS_TILE_SIZE + (blk & 1) * 8;
    const int by = (tile / tiles_x) * DARBS_TILE_SIZE + (blk >> 1) * 4;
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
    if (__reduce_max_sync(kFull, px.nproc) == 0) return;
    px.s = (px.g0 * bg0 + px.g1 * bg1 + px.g2 * bg2) * px.T;

    constexpr bool kPair = BwdExchange<FAM>::kPair;
    constexpr int kYzWords = kPair ? 2 : 1;  // floats per (pixel, entry) slot of the second array
    float4* gp = gpix[warp];
    float* xw = xch[warp][0];
    float* xyz = xch[warp][1];
    gp[lane] = make_float4(px.g0, px.g1, px.g2, 1.f);  // .w = 1 accumulates the weight sum

    // sweep-2 role of this lane: entry sj of the batch, pixels [16 sh, 16 sh + 16)
    const int sj = lane & (kBwdBatch - 1), sh = lane >> 4;
    const float* rw = xw + (sh * 16) * kXStride + sj;
    const float* ryz = xyz + kYzWords * ((sh * 16) * kXStride + sj);
    const float4* rg = gp + sh * 16;
    const float ex0 = X0, ey0 = Y0 + 2.f * sh;
    float* ww = xw + lane * kXStride;
    float* wyz = xyz + kYzWords * (lane * kXStride);

    // The entries the forward composited, [0, used), chunk by chunk from the last.  Entries of the
    // last batch beyond `used` (the stream is padded to a whole batch) and entries past the last
    // position a pixel processed are simply not eligible for that pixel.
    const float4* src = streams + kEntryVecs * stream_offset(tile, range.x, range.y, blk);
    const int used = stream_used[tile * kBlocksPerTile + blk];
    const int nchunks = (used + kChunk - 1) / kChunk;
    float4* stage0 = ring[warp][0];
    unsigned long long* bar = bars[warp];
    if (lane == 0) {
        for (int s = 0; s < kBwdStages; ++s) mbar_init(bar + s);
        mbar_init_fence();
        // the first kBwdStages - 1 chunks (from the back) in flight before the loop
        for (int s = 0; s < kBwdStages - 1; ++s)
            if (nchunks > s)
                bulk_load(stage0 + s * kChunkVecs, src + (size_t)(nchunks - 1 - s) * kChunkVecs, kChunkBytes, bar + s);
    }
    __syncwarp();
    int stage = 0;
    unsigned parity = 0;
    for (int c = nchunks - 1; c >= 0; --c) {
        if (lane == 0 && c >= kBwdStages - 1) {
            const int fill = stage == 0 ? kBwdStages - 1 : stage - 1;  // the stage chunk c + 1 vacated
            bulk_load(stage0 + fill * kChunkVecs, src + (size_t)(c - (kBwdStages - 1)) * kChunkVecs, kChunkBytes,
                      bar + fill);
        }
        mbar_wait(bar + stage, parity);
        const float4* qc = stage0 + stage * kChunkVecs;
        // entry `lane` of the chunk: can its alpha reach the clamp?  (bits of batches that do not run
        // may cover bytes beyond the stream's padding; they are not looked at)
        const unsigned clampable =
            FAM == FAM_GENERIC ? kFull : __ballot_sync(kFull, !(qc[lane * kEntryVecs + 1].y < kClampableF));
        const int first = used - c * kChunk > kBwdBatch ? 1 : 0;  // upper batch holds composited entries?
        for (int h = first; h >= 0; --h) {
            const float4* qb = qc + h * (kBwdBatch * kEntryVecs);
            // ---- sweep 1: lane = pixel, entries in descending list position
            for (int j0 = kBwdBatch - kBwdGroup; j0 >= 0; j0 -= kBwdGroup) {
                const BwdPixel save = px;
                bool near_acc = false;
                if ((clampable >> (h * kBwdBatch + j0)) & ((1u << kBwdGroup) - 1u)) {
#pragma unroll
                    for (int j = kBwdGroup - 1; j >= 0; --j)
                        bwd_visit<FAM, false, true>(kp, recs, qb + (j0 + j) * 3, fx, fy, px, ww + j0 + j,
                                                    wyz + kYzWords * (j0 + j), near_acc);
                } else {
#pragma unroll
                    for (int j = kBwdGroup - 1; j >= 0; --j)
                        bwd_visit<FAM, false, false>(kp, recs, qb + (j0 + j) * 3, fx, fy, px, ww + j0 + j,
                                                     wyz + kYzWords * (j0 + j), near_acc);
                }
                if (kp.exact && __any_sync(kFull, near_acc)) {  // a few groups per thousand
                    px = save;
                    for (int j = kBwdGroup - 1; j >= 0; --j)
                        bwd_visit<FAM, true, true>(kp, recs, qb + (j0 + j) * 3, fx, fy, px, ww + j0 + j,
                                                   wyz + kYzWords * (j0 + j), near_acc);
                }
            }
            __syncwarp();
            // ---- sweep 2: lane = (entry, half of the pixels)
            {
                const float4 r0 = qb[sj * 3 + 0];
                const float4 r1 = qb[sj * 3 + 1];
                const float4 r2 = qb[sj * 3 + 2];
                // packed FP32 (fma.rn.f32x2): two accumulators per instruction
                float2 dxy = make_float2(ex0 - r0.x, ey0 - r0.y);
                float2 dc01 = make_float2(0.f, 0.f), dc2w = dc01, sxxxy = dc01, sxsy = dc01;
                float syy = 0.f, dop = 0.f;
                const float2 step_x = make_float2(1.f, 0.f), step_row = make_float2(-7.f, 1.f);
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const float wv = rw[i * kXStride];
                    float yv, zv;
                    if constexpr (kPair) {
                        const float2 yz = *reinterpret_cast<const float2*>(ryz + 2 * i * kXStride);
                        yv = yz.x;
                        zv = yz.y;
                    } else {
                        yv = zv = ryz[i * kXStride];
                    }
                    const float4 g = rg[i];
                    const float2 wv2 = make_float2(wv, wv);
                    dc01 = __ffma2_rn(wv2, make_float2(g.x, g.y), dc01);
                    dc2w = __ffma2_rn(wv2, make_float2(g.z, g.w), dc2w);
                    const float2 zxy = __fmul2_rn(make_float2(zv, zv), dxy);  // z (dx, dy)
                    sxxxy = __ffma2_rn(make_float2(zxy.x, zxy.x), dxy, sxxxy);
                    sxsy = __fadd2_rn(sxsy, zxy);
                    syy = fmaf(zxy.y, dxy.y, syy);
                    dop += yv;
                    dxy = __fadd2_rn(dxy, (i & 7) == 7 ? step_row : step_x);
                }
                float dc0 = dc01.x, dc1 = dc01.y, dc2 = dc2w.x, wsum = dc2w.y;
                float sxx = sxxxy.x, sxy = sxxxy.y, sx = sxsy.x, sy = sxsy.y;
                // fold the two pixel halves (lanes l and l ^ 16 hold the same entry)
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
                if constexpr (!kPair) {  // the moments were taken of y: z = -ln2 o y
                    const float zs = -0.6931471805599453f * r1.y;
                    sxx *= zs;
                    sxy *= zs;
                    syy *= zs;
                    sx *= zs;
                    sy *= zs;
                }
                if (sh == 0 && wsum > 0.f) {
                    // SplatGrads order d_color[3], d_opacity, d_conic_a, d_conic_b, d_conic_c, d_mu2;
                    // m = scale * (a dx^2 + 2 b dx dy + c dy^2): dm/da = scale dx^2, dm/db = 2 scale dx dy,
                    // dm/d mu = -(2A dx + B dy, B dx + 2C dy) with (A, B, C) the scaled record values.
                    if constexpr (DET) {
                        long long* dst = reinterpret_cast<long long*>(grads) +
                                         (size_t)__float_as_int(r2.w) * DARBS_GRADS_PER_SPLAT;
                        fixed_add(dst + 0, dc0);
                        fixed_add(dst + 1, dc1);
                        fixed_add(dst + 2, dc2);
                        fixed_add(dst + 3, dop);
                        fixed_add(dst + 4, kp.scale * sxx);
                        fixed_add(dst + 5, 2.f * kp.scale * sxy);
                        fixed_add(dst + 6, kp.scale * syy);
                        fixed_add(dst + 7, -fmaf(2.f * r0.z, sx, r1.x * sy));
                        fixed_add(dst + 8, -fmaf(r1.x, sx, 2.f * r0.w * sy));
                    } else {
                        float* dst = grads + (size_t)__float_as_int(r2.w) * kSplatGradStride;
                        atomicAdd(reinterpret_cast<float4*>(dst), make_float4(dc0, dc1, dc2, dop));
                        atomicAdd(reinterpret_cast<float4*>(dst) + 1,
                                  make_float4(kp.scale * sxx, 2.f * kp.scale * sxy, kp.scale * syy,
                                              -fmaf(2.f * r0.z, sx, r1.x * sy)));
                        atomicAdd(dst + 8, -fmaf(r1.x, sx, 2.f * r0.w * sy));
                    }
                }
            }
            __syncwarp();
        }
        if (stage == kBwdStages - 1) {
            stage = 0;
            parity ^= 1u;
        } else {
            ++stage;
        }
    }
    const unsigned nexact = __reduce_add_sync(kFull, px.nexact);
    if (lane == 0 && nexact) atomicAdd(counters + CNT_EXACT, (unsigned long long)nexact);
}

// deterministic mode: int64 fixed-point sums (9 per splat) -> the padded float rows
__global__ void fixed_to_float_kernel(int64_t n, const long long* __restrict__ fx, float* __restrict__ padded) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n * kSplatGradStride) return;
    const int64_t row = i / kSplatGradStride;
    const int c = (int)(i - row * kSplatGradStride);
    padded[i] = c < DARBS_GRADS_PER_SPLAT ? (float)((double)fx[row * DARBS_GRADS_PER_SPLAT + c] * (1.0 / kFixedScale)) : 0.f;
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
            case FAM_MSINC1: eval_one_fast<FAM_MSINC1>(kp, x, wo, dwo); break;
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

// Tests every list entry against the eight blocks of its tile and writes the per-block
// survivor streams the render kernels consume.
// How many entries of a tile's list the cull kernel covers before the forward takes over block by
// block (forward_tail).  What a block needs is a saturation depth that belongs to the family, not to
// the list: measured (scratch/seg_sweep.py, cull + forward in us, segment -> time):
//   1 M splats 1080p   gaussian all 426, 512 484 | half-cosine-sq 256 222, all 290 |
//                      raised-cosine all 309, 384 343 | inv-multiquadric 256 260, all 335
//   3 M splats 4K      gaussian 384 1385, all 1866 | half-cosine-sq 128 710, 256 753, all 1661 |
//                      raised-cosine 384 1212, all 1348 | inv-multiquadric 192 822, 256 864, all 1949
// so: a base depth per family, applied when the mean list is at least 1.5 times as long (the tail
// path reads its entries from global memory and is slower per visit than the stream walk).
// ctx->cull_segment > 0 overrides (darbs_cuda_set_cull_segment).
// the CTA order of the render kernels: longest tile list first when this view's tile sort made one
static const int* tile_order_ptr(const darbs_cuda_ctx* ctx) {
    return ctx->tile_order_valid ? (const int*)ctx->tile_order.ptr : nullptr;
}

constexpr int kNoSegment = 1 << 30;
int cull_segment(const darbs_cuda_ctx* ctx, const KParams& kp) {
    if (ctx->cull_segment > 0) return ctx->cull_segment;
    const int base = (kp.fam == FAM_HCOS2 || kp.fam == FAM_IMQ) ? 256 : 384;
    const long long tiles = (long long)ctx->tiles_x * ctx->tiles_y;
    // with a promised capacity instead of K (darbs_cuda_set_entry_capacity) the host only knows the
    // bound; the promise is documented as 1.25 x the expected K
    const long long k = ctx->entry_capacity > 0 ? ctx->fwd_entries * 4 / 5 : ctx->fwd_entries;
    return (tiles > 0 && 2 * k >= 3 * (long long)base * tiles) ? base : kNoSegment;
}

darbs_status launch_cull(darbs_cuda_ctx* ctx, const KParams& kp) {
    const int tiles = ctx->tiles_x * ctx->tiles_y;
    if (tiles == 0) return DARBS_OK;
    const size_t k = (size_t)(ctx->fwd_entries > 0 ? ctx->fwd_entries : 0);
    const size_t entries = (size_t)kBlocksPerTile * (k + (size_t)kChunk * (size_t)tiles);
    DARBS_TRY(reserve(ctx, ctx->streams, sizeof(float4) * kEntryVecs * entries));
    DARBS_TRY(reserve(ctx, ctx->stream_count, sizeof(int) * 2 * kBlocksPerTile * (size_t)tiles));
    cull_kernel<<<tiles, kThreads, 0, ctx->stream>>>(
        kp, (const float4*)ctx->recs.ptr, (const int2*)ctx->ranges.ptr, point_list_ptr(ctx), ctx->tiles_x,
        cull_segment(ctx, kp), (float4*)ctx->streams.ptr, (int*)ctx->stream_count.ptr,
        (unsigned long long*)ctx->counters.ptr, nullptr);  // raster order: neighbouring tiles share records
    return check_launch(ctx, "cull_kernel");
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
    const int* count = (const int*)ctx->stream_count.ptr;
    int* used = (int*)ctx->stream_count.ptr + (size_t)kBlocksPerTile * tiles;
    const int seg = cull_segment(ctx, kp);
    if (ctx->tile_order_pending) {  // the ordering ran on the second stream, under the cull kernel
        DARBS_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, ctx->order_ready, 0));
        ctx->tile_order_pending = false;
    }
#define DARBS_LAUNCH_FWD_(F, T)                                                                      \
    render_fwd_kernel<F, T><<<tiles * (kBlocksPerTile / kFwdWarps), 32 * kFwdWarps, 0, ctx->stream>>>(  \
        kp, recs, ranges, plist, seg, (const float4*)ctx->streams.ptr, count, used, width, height,     \
        ctx->tiles_x, bg[0], bg[1], bg[2], image, t_final, processed, contributors, counters,          \
        tile_order_ptr(ctx))
#define DARBS_LAUNCH_FWD(F)              \
    do {                                 \
        if (seg < kNoSegment)            \
            DARBS_LAUNCH_FWD_(F, true);  \
        else                             \
            DARBS_LAUNCH_FWD_(F, false); \
    } while (0)
    switch (kp.fam) {
        case FAM_GAUSS2: DARBS_LAUNCH_FWD(FAM_GAUSS2); break;
        case FAM_HCOS2: DARBS_LAUNCH_FWD(FAM_HCOS2); break;
        case FAM_RCOS1: DARBS_LAUNCH_FWD(FAM_RCOS1); break;
        case FAM_IMQ: DARBS_LAUNCH_FWD(FAM_IMQ); break;
        case FAM_MSINC1: DARBS_LAUNCH_FWD(FAM_MSINC1); break;
        default: DARBS_LAUNCH_FWD(FAM_GENERIC); break;
    }
#undef DARBS_LAUNCH_FWD_
#undef DARBS_LAUNCH_FWD
    return check_launch(ctx, "render_fwd_kernel");
}

// Accumulates into ctx->splat_grads, n rows of kSplatGradStride floats (SplatGrads order in the
// first nine), zeroed here.
darbs_status launch_render_bwd(darbs_cuda_ctx* ctx, const KParams& kp, int width, int height,
                               const float bg[3], const float* grad_image, const float* t_final,
                               const int32_t* processed, int64_t n) {
    const size_t rows = (size_t)(n > 0 ? n : 1);
    const size_t bytes = sizeof(float) * kSplatGradStride * rows;
    const bool det = ctx->deterministic != 0;
    DARBS_TRY(reserve(ctx, ctx->splat_grads, bytes));
    float* sums = (float*)ctx->splat_grads.ptr;
    if (det) {
        const size_t fx_bytes = sizeof(long long) * DARBS_GRADS_PER_SPLAT * rows;
        DARBS_TRY(reserve(ctx, ctx->splat_grads_fx, fx_bytes));
        DARBS_CUDA_TRY(ctx, cudaMemsetAsync(ctx->splat_grads_fx.ptr, 0, fx_bytes, ctx->stream));
        sums = (float*)ctx->splat_grads_fx.ptr;
    }
    int tiles = ctx->tiles_x * ctx->tiles_y;
    if (!det || tiles == 0 || n == 0)
        DARBS_CUDA_TRY(ctx, cudaMemsetAsync(ctx->splat_grads.ptr, 0, bytes, ctx->stream));
    if (tiles == 0 || n == 0) return DARBS_OK;
    auto* counters = (unsigned long long*)ctx->counters.ptr;
    const float4* recs = (const float4*)ctx->recs.ptr;
    const int2* ranges = (const int2*)ctx->ranges.ptr;
    const int* used = (const int*)ctx->stream_count.ptr + (size_t)kBlocksPerTile * tiles;
#define DARBS_LAUNCH_BWD_(F, D)                                                                   \
    render_bwd_kernel<F, D><<<tiles * (kBlocksPerTile / kBwdWarps), kBwdThreads, 0, ctx->stream>>>(  \
        kp, recs, ranges, (const float4*)ctx->streams.ptr, used, width, height, ctx->tiles_x,     \
        bg[0], bg[1], bg[2], grad_image, t_final, processed, sums, counters, tile_order_ptr(ctx))
#define DARBS_LAUNCH_BWD(F)              \
    do {                                 \
        if (det)                         \
            DARBS_LAUNCH_BWD_(F, true);  \
        else                             \
            DARBS_LAUNCH_BWD_(F, false); \
    } while (0)
    switch (kp.fam) {
        case FAM_GAUSS2: DARBS_LAUNCH_BWD(FAM_GAUSS2); break;
        case FAM_HCOS2: DARBS_LAUNCH_BWD(FAM_HCOS2); break;
        case FAM_RCOS1: DARBS_LAUNCH_BWD(FAM_RCOS1); break;
        case FAM_IMQ: DARBS_LAUNCH_BWD(FAM_IMQ); break;
        case FAM_MSINC1: DARBS_LAUNCH_BWD(FAM_MSINC1); break;
        default: DARBS_LAUNCH_BWD(FAM_GENERIC); break;
    }
#undef DARBS_LAUNCH_BWD
#undef DARBS_LAUNCH_BWD_
    DARBS_TRY(check_launch(ctx, "render_bwd_kernel"));
    if (det) {
        const int64_t count = n * kSplatGradStride;
        fixed_to_float_kernel<<<(unsigned)((count + 255) / 256), 256, 0, ctx->stream>>>(
            n, (const long long*)ctx->splat_grads_fx.ptr, (float*)ctx->splat_grads.ptr);
        DARBS_TRY(check_launch(ctx, "fixed_to_float_kernel"));
    }
    return DARBS_OK;
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
