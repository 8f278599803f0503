// loss.cu — L = (1 - lambda) L1 + lambda (1 - SSIM)/2 and dL/d(rendered image) on the device.
//
// Reference: darbs::loss_total src/loss.cpp:173-230 (window :13-32, mirror padding :35-41,
// separable moment filters :47-74, their adjoints :76-115, ssim_terms :124-140).
//
// Images are row-major RGB interleaved, so a row is a plane of 3w floats in which the window's
// taps sit three floats apart; all three channels are processed at once and every global access
// is a contiguous run.  A CTA of 128 threads owns a tile of 32 x 16 pixels:
//
//   phase 1 (columns)  thread = one of the 126 float columns of the tile plus its halo; it walks
//                      the 26 input rows once (mirror-reflected row / pixel indices for the
//                      moments, zero extension for the adjoint), forms the products once per
//                      element and feeds 16 register accumulators per quantity: 11 FMAs per
//                      output and quantity, no halo recomputation, packed two quantities to an
//                      instruction (fma.rn.f32x2).  Results go to shared memory.
//   phase 2 (rows)     thread = (row, group of 4 pixels): 42 consecutive shared-memory floats
//                      per quantity feed 12 outputs, again 11 packed FMAs each.
//
//   ssim_map_kernel    windowed moments of x = rendered and d = rendered - target, the SSIM
//                      partials (below) scaled by -lambda / (2 n) into three maps, and the sums
//                      of |d|, d^2 and 1 - SSIM.
//   ssim_grad_kernel   the adjoint window over the zero-extended maps, then
//                      grad = (1 - lambda) sign(d)/n + s_a + x s_e - d s_d, for pixels at least
//                      five away from every edge.
//   (border CTAs)      pixels within five of an edge, where mirror padding folds taps back
//                      (loss.cpp:35-41, :76-103): the adjoint weights are enumerated exactly
//                      with reflect().  Handles images smaller than the window too.  They are
//                      the first CTAs of the ssim_grad_kernel launch, so they run under the
//                      interior tiles.
//
// Numerics (FP32 against the FP64 reference).  The reference's three partials d/d mu_x,
// d/d s_xx, d/d s_xy (loss.cpp:133-138) and its combination s_a + 2 x s_b + y s_d (:222-224)
// cancel catastrophically when the images are close, which is where training spends its time.
// The same quantities are therefore written in the small differences themselves: with
// d = x - y, m = mu_d^2 = b1 - a1, v = var_d = b2 - a2 (moments of d are filtered directly),
//   1 - S   = (a1 v + a2 m + m v) / (b1 b2)
//   f_a     = [2 (a2 - a1) (mu_x (1 - S) - mu_d) - 2 mu_x S (v - m)] / (b1 b2)     (= d/d mu_x)
//   f_e     = 2 a1 v / (b1 b2^2)                                       (= 2 d/d s_xx + d/d s_xy)
//   f_d     = 2 a1 / (b1 b2)                                                       (= d/d s_xy)
//   grad   += s_a + x s_e - d s_d          (2 x s_b + y s_d = x (2 s_b + s_d) - d s_d)
// and every term vanishes by itself as y -> x.  Moments are accumulated on values shifted by a
// per-tile, per-channel reference (the tile's centre pixel); variances are shift invariant.
#include "common.cuh"

namespace darbs_b200 {

namespace {

constexpr int kWin = 11, kHalf = 5;
#ifndef DARBS_LOSS_TH
#define DARBS_LOSS_TH 16
#endif
#ifndef DARBS_LOSS_PX
#define DARBS_LOSS_PX 4
#endif
#ifndef DARBS_LOSS_MINB
#define DARBS_LOSS_MINB 5
#endif
#ifndef DARBS_LOSS_AHEAD
#define DARBS_LOSS_AHEAD 4
#endif
constexpr int kTW = 32, kTH = DARBS_LOSS_TH;   // tile, pixels
constexpr int kCols = 3 * (kTW + 2 * kHalf);   // 126 float columns with halo
constexpr int kRowsIn = kTH + 2 * kHalf;       // input rows
constexpr int kPX = DARBS_LOSS_PX;             // pixels per phase-2 thread
constexpr int kGroups = kTW / kPX;             // phase-2 threads per tile row
constexpr int kOut = 3 * kPX;                  // floats per phase-2 thread: kPX pixels x 3 channels
constexpr int kSpan = kOut + 3 * (kWin - 1);   // floats that feed them
constexpr int kLossThreads = 128;
constexpr int kAhead = DARBS_LOSS_AHEAD;        // rows of global loads in flight per thread in the column passes
static_assert(kLossThreads >= kCols && kLossThreads == kTH * kGroups, "thread mapping");
static_assert(kPX == 4 || kPX == 2, "vector width of the row accesses");

struct Window {
    float k[kWin];
};

Window make_window() {  // loss.cpp:19-32
    double w[kWin], sum = 0.0;
    for (int i = 0; i < kWin; ++i) {
        double d = i - kHalf;
        w[i] = exp(-d * d / (2.0 * 1.5 * 1.5));
        sum += w[i];
    }
    Window out;
    for (int i = 0; i < kWin; ++i) out.k[i] = (float)(w[i] / sum);
    return out;
}

__device__ __forceinline__ int reflect(int i, int n) {  // loss.cpp:35-41
    while (i < 0 || i >= n) {
        if (i < 0) i = -i - 1;
        if (i >= n) i = 2 * n - 1 - i;
    }
    return i;
}

__device__ __forceinline__ float2 fma2(float k, float2 p, float2 acc) {
    return __ffma2_rn(make_float2(k, k), p, acc);
}

__device__ __forceinline__ void block_sum3(float a, float b, float c, double* __restrict__ sums, int fixed) {
    __shared__ double red[3][kLossThreads / 32];
    double d0 = a, d1 = b, d2 = c;
    for (int o = 16; o > 0; o >>= 1) {
        d0 += __shfl_xor_sync(0xffffffffu, d0, o);
        d1 += __shfl_xor_sync(0xffffffffu, d1, o);
        d2 += __shfl_xor_sync(0xffffffffu, d2, o);
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = d0;
        red[1][threadIdx.x >> 5] = d1;
        red[2][threadIdx.x >> 5] = d2;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        double t = 0.0;
        for (int w = 0; w < kLossThreads / 32; ++w) t += red[threadIdx.x][w];
        if (fixed)  // deterministic mode: order-independent int64 fixed point in the same slot
            atomicAdd(reinterpret_cast<unsigned long long*>(sums) + threadIdx.x,
                      (unsigned long long)__double2ll_rn(t * kFixedScale));
        else
            atomicAdd(sums + threadIdx.x, t);
    }
}

// kOut consecutive floats of a row, as three 128-bit (kPX = 4) or 64-bit (kPX = 2) accesses when
// the row is 16-byte aligned
template <bool VEC>
__device__ __forceinline__ void load12(const float* __restrict__ p, int valid, float out[kOut]) {
    if constexpr (VEC && kPX == 4) {
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(p) + q);
            out[4 * q + 0] = v.x;
            out[4 * q + 1] = v.y;
            out[4 * q + 2] = v.z;
            out[4 * q + 3] = v.w;
        }
    } else if constexpr (VEC) {
#pragma unroll
        for (int q = 0; q < kOut / 2; ++q) {
            const float2 v = __ldg(reinterpret_cast<const float2*>(p) + q);
            out[2 * q + 0] = v.x;
            out[2 * q + 1] = v.y;
        }
    } else {
#pragma unroll
        for (int e = 0; e < kOut; ++e) out[e] = e < valid ? __ldg(p + e) : 0.f;
    }
}

template <bool VEC>
__device__ __forceinline__ void store12(float* __restrict__ p, int valid, const float v[kOut]) {
    if constexpr (VEC && kPX == 4) {
#pragma unroll
        for (int q = 0; q < 3; ++q)
            reinterpret_cast<float4*>(p)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    } else if constexpr (VEC) {
#pragma unroll
        for (int q = 0; q < kOut / 2; ++q) reinterpret_cast<float2*>(p)[q] = make_float2(v[2 * q], v[2 * q + 1]);
    } else {
#pragma unroll
        for (int e = 0; e < kOut; ++e)
            if (e < valid) p[e] = v[e];
    }
}

// ---------------------------------------------------------------- moments + SSIM partials
template <bool VEC>
__global__ void __launch_bounds__(kLossThreads, DARBS_LOSS_MINB)
ssim_map_kernel(Window win, int w, int h, const float* __restrict__ image,
                const float* __restrict__ target, float scale, int want_maps,
                float* __restrict__ fa, float* __restrict__ fe, float* __restrict__ fd,
                double* __restrict__ sums, int fixed) {
    __shared__ float2 s_v01[kTH * kCols];  // (sum k x', sum k d')
    __shared__ float2 s_v23[kTH * kCols];  // (sum k x'^2, sum k d'^2)
    __shared__ float s_v4[kTH * kCols];    //  sum k x' d'
    __shared__ int s_row[kRowsIn];  // element offset of each (mirror-reflected) input row
    __shared__ float s_ref[2][3];
    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * kTW, y0 = blockIdx.y * kTH;
    if (tid < kRowsIn) s_row[tid] = reflect(y0 - kHalf + tid, h) * w * 3;
    if (tid < 3) {
        const size_t p = ((size_t)min(y0 + kTH / 2, h - 1) * w + min(x0 + kTW / 2, w - 1)) * 3 + tid;
        const float rx = __ldg(image + p);
        s_ref[0][tid] = rx;
        s_ref[1][tid] = rx - __ldg(target + p);
    }
    __syncthreads();
    // ---- phase 1: columns (filter_y, loss.cpp:62-74, applied first: the two passes commute)
    if (tid < kCols) {
        const int ch = tid % 3;
        const int gx = reflect(x0 - kHalf + tid / 3, w);
        const float* ip = image + (size_t)gx * 3 + ch;
        const float* tp = target + (size_t)gx * 3 + ch;
        const float refx = s_ref[0][ch], refd = s_ref[1][ch];
        float2 a01[kTH], a23[kTH];
        float a4[kTH];
#pragma unroll
        for (int o = 0; o < kTH; ++o) {
            a01[o] = a23[o] = make_float2(0.f, 0.f);
            a4[o] = 0.f;
        }
        // the rows are requested kAhead iterations before their use: a warp's walk down its columns
        // is otherwise one dependent global load per row (measured: the kernel's long-scoreboard stalls)
        float xq[kAhead], tq[kAhead];
#pragma unroll
        for (int i = 0; i < kAhead && i < kRowsIn; ++i) {
            xq[i] = __ldg(ip + s_row[i]);
            tq[i] = __ldg(tp + s_row[i]);
        }
#pragma unroll
        for (int i = 0; i < kRowsIn; ++i) {
            const float xv = xq[i % kAhead], tv = tq[i % kAhead];
            if (i + kAhead < kRowsIn) {
                xq[i % kAhead] = __ldg(ip + s_row[i + kAhead]);
                tq[i % kAhead] = __ldg(tp + s_row[i + kAhead]);
            }
            const float xs = xv - refx, ds = (xv - tv) - refd;
            const float2 p01 = make_float2(xs, ds), p23 = make_float2(xs * xs, ds * ds);
            const float p4 = xs * ds;
#pragma unroll
            for (int o = 0; o < kTH; ++o) {
                const int t = i - o;
                if (t >= 0 && t < kWin) {
                    a01[o] = fma2(win.k[t], p01, a01[o]);
                    a23[o] = fma2(win.k[t], p23, a23[o]);
                    a4[o] = fmaf(win.k[t], p4, a4[o]);
                }
            }
        }
#pragma unroll
        for (int o = 0; o < kTH; ++o) {
            s_v01[o * kCols + tid] = a01[o];
            s_v23[o * kCols + tid] = a23[o];
            s_v4[o * kCols + tid] = a4[o];
        }
    }
    __syncthreads();
    // ---- phase 2: rows (filter_x, loss.cpp:47-60) and ssim_terms (loss.cpp:124-140)
    const int o = tid / kGroups, g = tid % kGroups;
    const int gy = y0 + o, gx0 = x0 + kPX * g;
    float sum_abs = 0.f, sum_sq = 0.f, sum_dssim = 0.f;
    if (gy < h && gx0 < w) {
        float2 r01[kOut], r23[kOut];
        float r4[kOut];
        {
            const float2* src = s_v01 + o * kCols + kOut * g;
            float2 v[kSpan];
#pragma unroll
            for (int j = 0; j < kSpan; ++j) v[j] = src[j];
#pragma unroll
            for (int e = 0; e < kOut; ++e) {
                float2 acc = make_float2(0.f, 0.f);
#pragma unroll
                for (int t = 0; t < kWin; ++t) acc = fma2(win.k[t], v[e + 3 * t], acc);
                r01[e] = acc;
            }
        }
        {
            const float2* src = s_v23 + o * kCols + kOut * g;
            float2 v[kSpan];
#pragma unroll
            for (int j = 0; j < kSpan; ++j) v[j] = src[j];
#pragma unroll
            for (int e = 0; e < kOut; ++e) {
                float2 acc = make_float2(0.f, 0.f);
#pragma unroll
                for (int t = 0; t < kWin; ++t) acc = fma2(win.k[t], v[e + 3 * t], acc);
                r23[e] = acc;
            }
        }
        {
            const float* src = s_v4 + o * kCols + kOut * g;
            float v[kSpan];
#pragma unroll
            for (int j = 0; j < kSpan; ++j) v[j] = src[j];
#pragma unroll
            for (int e = 0; e < kOut; ++e) {
                float acc = 0.f;
#pragma unroll
                for (int t = 0; t < kWin; ++t) acc = fmaf(win.k[t], v[e + 3 * t], acc);
                r4[e] = acc;
            }
        }
        const int valid = 3 * min(kPX, w - gx0);
        const size_t p = ((size_t)gy * w + gx0) * 3;
        float xc[kOut], yc[kOut];
        load12<VEC>(image + p, valid, xc);
        load12<VEC>(target + p, valid, yc);
        float oa[kOut], oe[kOut], od[kOut];
        const float c1 = 0.01f * 0.01f, c2 = 0.03f * 0.03f;
#pragma unroll
        for (int e = 0; e < kOut; ++e) {
            const int ch = e % 3;
            const float mxs = r01[e].x, mds = r01[e].y;
            const float mu_x = mxs + s_ref[0][ch], mu_d = mds + s_ref[1][ch];
            const float mu_y = mu_x - mu_d;
            const float var_x = r23[e].x - mxs * mxs;
            const float v = fmaxf(r23[e].y - mds * mds, 0.f);  // var_d = b2 - a2
            const float cov_xd = r4[e] - mxs * mds;
            const float m = mu_d * mu_d;                        // b1 - a1
            const float a1 = 2.f * mu_x * mu_y + c1;
            const float a2 = 2.f * (var_x - cov_xd) + c2;       // 2 cov_xy + C2
            const float b1 = a1 + m, b2 = a2 + v;
            float inv_b1, inv_b2;  // b1 >= C1, b2 >= C2: one MUFU each, 1 ulp
            asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv_b1) : "f"(b1));
            asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv_b2) : "f"(b2));
            const float inv = inv_b1 * inv_b2;
            const float one_minus_s = (a1 * v + a2 * m + m * v) * inv;
            const float s = 1.0f - one_minus_s;
            const float d = xc[e] - yc[e];  // 0 past `valid` (load12)
            sum_dssim += (VEC || e < valid) ? one_minus_s : 0.f;
            sum_abs += fabsf(d);
            sum_sq = fmaf(d, d, sum_sq);
            const float na = 2.f * (a2 - a1) * (mu_x * one_minus_s - mu_d) - 2.f * mu_x * s * (v - m);
            oa[e] = scale * na * inv;
            oe[e] = scale * 2.f * a1 * v * inv * inv_b2;
            od[e] = scale * 2.f * a1 * inv;
        }
        if (want_maps) {
            store12<VEC>(fa + p, valid, oa);
            store12<VEC>(fe + p, valid, oe);
            store12<VEC>(fd + p, valid, od);
        }
    }
    block_sum3(sum_abs, sum_sq, sum_dssim, sums, fixed);
}

// ---------------------------------------------------------------- adjoint, interior pixels
template <bool VEC>
__device__ __forceinline__ void grad_interior_tile(const Window& win, int w, int h, int tile_x, int tile_y,
                                                   const float* __restrict__ image,
                                                   const float* __restrict__ target, const float* __restrict__ fa,
                                                   const float* __restrict__ fe, const float* __restrict__ fd,
                                                   float coef_l1, float* __restrict__ grad) {
    __shared__ float2 s_v01[kTH * kCols];  // columns pass of (f_a, f_e)
    __shared__ float s_v2[kTH * kCols];    // columns pass of f_d
    __shared__ int s_row[kRowsIn];         // element offset of each input row, -1 outside the image
    const int tid = threadIdx.x;
    const int x0 = tile_x * kTW, y0 = tile_y * kTH;
    if (tid < kRowsIn) {
        const int gy = y0 - kHalf + tid;
        s_row[tid] = gy >= 0 && gy < h ? gy * w * 3 : -1;
    }
    __syncthreads();
    // ---- phase 1: columns (scatter_y, loss.cpp:91-103, as a gather over the zero-extended map)
    if (tid < kCols) {
        const int gx = x0 - kHalf + tid / 3;
        const bool col_in = gx >= 0 && gx < w;
        const int cbase = col_in ? gx * 3 + tid % 3 : 0;
        float2 a01[kTH];
        float a2[kTH];
#pragma unroll
        for (int o = 0; o < kTH; ++o) {
            a01[o] = make_float2(0.f, 0.f);
            a2[o] = 0.f;
        }
        float aq[kAhead], eq[kAhead], dq[kAhead];  // rows requested kAhead iterations ahead, as in ssim_map_kernel
        auto fetch = [&](int i, float& a, float& e, float& d) {
            const int roff = s_row[i];
            const bool in = col_in && roff >= 0;
            const int p = in ? roff + cbase : 0;
            a = in ? __ldg(fa + p) : 0.f;
            e = in ? __ldg(fe + p) : 0.f;
            d = in ? __ldg(fd + p) : 0.f;
        };
#pragma unroll
        for (int i = 0; i < kAhead && i < kRowsIn; ++i) fetch(i, aq[i], eq[i], dq[i]);
#pragma unroll
        for (int i = 0; i < kRowsIn; ++i) {
            const float2 p01 = make_float2(aq[i % kAhead], eq[i % kAhead]);
            const float p2 = dq[i % kAhead];
            if (i + kAhead < kRowsIn) fetch(i + kAhead, aq[i % kAhead], eq[i % kAhead], dq[i % kAhead]);
#pragma unroll
            for (int o = 0; o < kTH; ++o) {
                const int t = i - o;
                if (t >= 0 && t < kWin) {
                    a01[o] = fma2(win.k[t], p01, a01[o]);
                    a2[o] = fmaf(win.k[t], p2, a2[o]);
                }
            }
        }
#pragma unroll
        for (int o = 0; o < kTH; ++o) {
            s_v01[o * kCols + tid] = a01[o];
            s_v2[o * kCols + tid] = a2[o];
        }
    }
    __syncthreads();
    // ---- phase 2: rows (scatter_x, loss.cpp:76-89) and the combination (loss.cpp:186, :222-224)
    const int o = tid / kGroups, g = tid % kGroups;
    const int gy = y0 + o, gx0 = x0 + kPX * g;
    if (gy < kHalf || gy >= h - kHalf || gx0 >= w - kHalf || gx0 + kPX - 1 < kHalf) return;  // border kernel's
    float2 r01[kOut];
    float r2[kOut];
    {
        const float2* src = s_v01 + o * kCols + kOut * g;
        float2 v[kSpan];
#pragma unroll
        for (int j = 0; j < kSpan; ++j) v[j] = src[j];
#pragma unroll
        for (int e = 0; e < kOut; ++e) {
            float2 acc = make_float2(0.f, 0.f);
#pragma unroll
            for (int t = 0; t < kWin; ++t) acc = fma2(win.k[t], v[e + 3 * t], acc);
            r01[e] = acc;
        }
    }
    {
        const float* src = s_v2 + o * kCols + kOut * g;
        float v[kSpan];
#pragma unroll
        for (int j = 0; j < kSpan; ++j) v[j] = src[j];
#pragma unroll
        for (int e = 0; e < kOut; ++e) {
            float acc = 0.f;
#pragma unroll
            for (int t = 0; t < kWin; ++t) acc = fmaf(win.k[t], v[e + 3 * t], acc);
            r2[e] = acc;
        }
    }
    const int valid = 3 * min(kPX, w - gx0);
    const size_t p = ((size_t)gy * w + gx0) * 3;
    float xc[kOut], yc[kOut], out[kOut];
    load12<VEC>(image + p, valid, xc);
    load12<VEC>(target + p, valid, yc);
#pragma unroll
    for (int e = 0; e < kOut; ++e) {
        const float d = xc[e] - yc[e];
        out[e] = coef_l1 * (float)((d > 0.f) - (d < 0.f)) + r01[e].x + xc[e] * r01[e].y - d * r2[e];
    }
    // the group may straddle the five-pixel band on the left or right
    const bool whole = gx0 >= kHalf && gx0 + kPX - 1 < w - kHalf;
    if (whole) {
        store12<VEC>(grad + p, valid, out);
    } else {
#pragma unroll
        for (int e = 0; e < kOut; ++e) {
            const int gx = gx0 + e / 3;
            if (gx >= kHalf && gx < w - kHalf) grad[p + e] = out[e];
        }
    }
}

// ---------------------------------------------------------------- adjoint, border pixels
// Pixels with x < 5, x >= w - 5, y < 5 or y >= h - 5: `top` full rows, `bottom` full rows, and
// `left` + `right` columns of the rows between them.  Eight lanes per pixel, three channels.
// The weight with which source i reaches position j along an axis of length n is
// sum_d k[d] [reflect(i + d) == j] (loss.cpp:76-103); every source of a border position lies
// within five of it (also after repeated reflection in images narrower than the window).
__device__ __forceinline__ float adjoint_weight(const Window& win, int i, int j, int n) {
    if (i < 0 || i >= n) return 0.f;
    float acc = 0.f;
    if (n >= 2 * kHalf) {
        // one reflection at most: position p = i + d lands on j directly, through the left edge
        // (p = -j - 1) or through the right edge (p = 2n - 1 - j)
        const int d0 = j - i, d1 = -j - 1 - i, d2 = 2 * n - 1 - j - i;
        if (d0 >= -kHalf && d0 <= kHalf) acc += win.k[d0 + kHalf];
        if (d1 >= -kHalf && d1 <= kHalf) acc += win.k[d1 + kHalf];
        if (d2 >= -kHalf && d2 <= kHalf) acc += win.k[d2 + kHalf];
    } else {
        for (int d = -kHalf; d <= kHalf; ++d)
            if (reflect(i + d, n) == j) acc += win.k[d + kHalf];
    }
    return acc;
}

constexpr int kBorderThreads = 128, kBorderLanes = 8;  // eight lanes share a pixel's 121 sources (measured faster than 32)

struct BorderBand {
    int top, bottom, left, right, count, blocks, stride;
};

__device__ __forceinline__ void grad_border_group(const Window& win, int w, int h, const BorderBand& band,
                                                  int group, const float* __restrict__ image,
                                                  const float* __restrict__ target, const float* __restrict__ fa,
                                                  const float* __restrict__ fe, const float* __restrict__ fd,
                                                  float coef_l1, float* __restrict__ grad) {
    __shared__ float s_w[kBorderThreads / kBorderLanes][2][kWin + 1];
    const int top = band.top, bottom = band.bottom, left = band.left, right = band.right, count = band.count;
    const int slot = threadIdx.x / kBorderLanes, sub = threadIdx.x % kBorderLanes;
    const int idx = group * (kBorderThreads / kBorderLanes) + slot;
    const bool active = idx < count;
    int x = 0, y = 0;
    if (active) {
        if (idx < top * w) {
            y = idx / w;
            x = idx - y * w;
        } else if (idx < (top + bottom) * w) {
            const int r = idx - top * w;
            y = h - bottom + r / w;
            x = r % w;
        } else {
            const int r = idx - (top + bottom) * w, side = left + right;
            y = top + r / side;
            const int c = r % side;
            x = c < left ? c : w - right + (c - left);
        }
        for (int s = sub; s < kWin; s += kBorderLanes) {
            s_w[slot][0][s] = adjoint_weight(win, y - kHalf + s, y, h);
            s_w[slot][1][s] = adjoint_weight(win, x - kHalf + s, x, w);
        }
    }
    __syncwarp();
    float acc[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (active) {
        for (int q = sub; q < kWin * kWin; q += kBorderLanes) {
            const int sy = q / kWin, sx = q - sy * kWin;
            const float wgt = s_w[slot][0][sy] * s_w[slot][1][sx];
            if (wgt == 0.f) continue;
            const size_t p = ((size_t)(y - kHalf + sy) * w + (x - kHalf + sx)) * 3;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                acc[c] = fmaf(wgt, __ldg(fa + p + c), acc[c]);
                acc[3 + c] = fmaf(wgt, __ldg(fe + p + c), acc[3 + c]);
                acc[6 + c] = fmaf(wgt, __ldg(fd + p + c), acc[6 + c]);
            }
        }
    }
#pragma unroll
    for (int v = 0; v < 9; ++v)
        for (int o = kBorderLanes / 2; o > 0; o >>= 1) acc[v] += __shfl_xor_sync(0xffffffffu, acc[v], o);
    if (active && sub < 3) {
        const int c = sub;
        const size_t p = ((size_t)y * w + x) * 3 + c;
        const float xv = __ldg(image + p), d = xv - __ldg(target + p);
        const float sa = c == 0 ? acc[0] : c == 1 ? acc[1] : acc[2];
        const float se = c == 0 ? acc[3] : c == 1 ? acc[4] : acc[5];
        const float sd = c == 0 ? acc[6] : c == 1 ? acc[7] : acc[8];
        grad[p] = coef_l1 * (float)((d > 0.f) - (d < 0.f)) + sa + xv * se - d * sd;
    }
}

// One launch for the whole adjoint: band.blocks CTAs, spread evenly over the grid, take the border
// pixels (latency bound: 121 scattered sources per pixel), the others one interior tile each, so
// the border work runs under the interior tiles instead of after them.
static_assert(kBorderThreads == kLossThreads, "one CTA shape for both roles");
template <bool VEC>
__global__ void __launch_bounds__(kLossThreads)
ssim_grad_kernel(Window win, int w, int h, BorderBand band, int tiles_x, const float* __restrict__ image,
                 const float* __restrict__ target, const float* __restrict__ fa,
                 const float* __restrict__ fe, const float* __restrict__ fd, float coef_l1,
                 float* __restrict__ grad) {
    // every band.stride-th CTA is a border one until they are used up
    const int b = blockIdx.x, q = b / band.stride;
    if (b - q * band.stride == 0 && q < band.blocks) {
        grad_border_group(win, w, h, band, q, image, target, fa, fe, fd, coef_l1, grad);
    } else {
        const int t = b - min(q + 1, band.blocks);
        grad_interior_tile<VEC>(win, w, h, t % tiles_x, t / tiles_x, image, target, fa, fe, fd, coef_l1, grad);
    }
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

}  // namespace

// loss_total (loss.cpp:173-230) on device arrays.  sums (device, 3 doubles, zeroed here) receive
// sum |d|, sum d^2 and sum (1 - SSIM); grad_image may be NULL (values only).
darbs_status launch_loss(darbs_cuda_ctx* ctx, int width, int height, const float* image,
                         const float* target, double lambda, float* grad_image, double* sums) {
    DARBS_CUDA_TRY(ctx, cudaMemsetAsync(sums, 0, sizeof(double) * 3, ctx->stream));
    const size_t px = (size_t)width * height;
    if (px == 0) return DARBS_OK;
    const int64_t count = (int64_t)(3 * px);
    static const Window win = make_window();
    const dim3 grid((unsigned)((width + kTW - 1) / kTW), (unsigned)((height + kTH - 1) / kTH));
    const bool maps = lambda != 0.0 && grad_image != nullptr;
    float *fa = nullptr, *fe = nullptr, *fd = nullptr;
    if (maps) {
        DARBS_TRY(reserve(ctx, ctx->loss_maps, sizeof(float) * 9 * px + 64));
        fa = (float*)ctx->loss_maps.ptr;
        fe = fa + ((3 * px + 3) & ~(size_t)3);
        fd = fe + ((3 * px + 3) & ~(size_t)3);
    }
    // 128-bit row accesses need every row to start 16-byte aligned: 3 w floats per row
    const int vec = (width % 4 == 0) && aligned16(image) && aligned16(target) && (!grad_image || aligned16(grad_image));
    const float scale = (float)(-0.5 * lambda / (double)count);  // loss.cpp:196
    if (count >= (int64_t)1 << 31) return fail(ctx, DARBS_INVALID_PARAMETER, "loss_total: image too large");
    if (vec)
        ssim_map_kernel<true><<<grid, kLossThreads, 0, ctx->stream>>>(win, width, height, image, target, scale,
                                                                      maps ? 1 : 0, fa, fe, fd, sums, ctx->deterministic);
    else
        ssim_map_kernel<false><<<grid, kLossThreads, 0, ctx->stream>>>(win, width, height, image, target, scale,
                                                                       maps ? 1 : 0, fa, fe, fd, sums, ctx->deterministic);
    DARBS_TRY(check_launch(ctx, "ssim_map_kernel"));
    if (!grad_image) return DARBS_OK;
    if (!maps) {
        // lambda == 0: the L1 gradient in one streaming pass; its |d|, d^2 sums go to a scratch pair
        return launch_l1_loss(ctx, count, image, target, 0.0, grad_image, sums + 3);
    }
    const float coef = (float)((1.0 - lambda) / (double)count);  // loss.cpp:186
    BorderBand band;
    band.top = height < kHalf ? height : kHalf;
    band.bottom = height - band.top < kHalf ? height - band.top : kHalf;
    const int middle = height - band.top - band.bottom;
    band.left = width < kHalf ? width : kHalf;
    band.right = width - band.left < kHalf ? width - band.left : kHalf;
    const long long border = (long long)(band.top + band.bottom) * width + (long long)middle * (band.left + band.right);
    const int per_block = kBorderThreads / kBorderLanes;
    band.count = (int)border;
    band.blocks = (int)((border + per_block - 1) / per_block);
    // interior tiles exist only when some pixel is five or more from every edge
    const bool interior = width > 2 * kHalf && height > 2 * kHalf;
    const unsigned blocks = (unsigned)band.blocks + (interior ? grid.x * grid.y : 0u);
    band.stride = band.blocks ? (int)(blocks / (unsigned)band.blocks) : 1;
    if (blocks) {
        if (vec)
            ssim_grad_kernel<true><<<blocks, kLossThreads, 0, ctx->stream>>>(win, width, height, band, (int)grid.x, image,
                                                                             target, fa, fe, fd, coef, grad_image);
        else
            ssim_grad_kernel<false><<<blocks, kLossThreads, 0, ctx->stream>>>(win, width, height, band, (int)grid.x, image,
                                                                              target, fa, fe, fd, coef, grad_image);
        DARBS_TRY(check_launch(ctx, "ssim_grad_kernel"));
    }
    return DARBS_OK;
}

}  // namespace darbs_b200
