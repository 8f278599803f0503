// splat.cuh — per-splat device helpers shared by the stand-alone kernels (rect_kernel,
// pack_kernel) and by the preprocess kernel of the training step, which fuses them:
//   tile rectangle + tile count   src/rasterizer.cpp:39-45
//   depth sort key                src/rasterizer.cpp:31-35 (order-preserving bit map)
//   packed 64-byte record         csrc/common.cuh (kRecVecs)
// Both paths evaluate them on the float32 splat values, so they produce identical bits.
#pragma once

#include "family.cuh"

namespace darbs_b200 {

__device__ __forceinline__ unsigned depth_to_key(float d) {
    // order-preserving map float -> uint (negative depths included)
    unsigned u = __float_as_uint(d);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// rect packed as x0 | y0<<16 and x1 | y1<<16 ; count == 0 -> no tiles.  `ok` = the splat exists
// for this view (not near-plane culled).
__device__ __forceinline__ void splat_rect(bool ok, float mxf, float myf, float a, float b, float c, float r,
                                           int tiles_x, int tiles_y, unsigned long long* skipped,
                                           uint2& rect, unsigned& cnt) {
    cnt = 0;
    rect = make_uint2(0, 0);
    if (!ok) return;
    if (!(isfinite(a) && isfinite(b) && isfinite(c) && isfinite(r))) {  // rasterizer.cpp:39
        atomicAdd(skipped, 1ull);
        return;
    }
    double mx = mxf, my = myf, rd = r;
    // rasterizer.cpp:40-45 (the clamp happens in floating point here so
    // that huge coordinates cannot overflow the int conversion)
    double fx0 = floor((mx - rd) / DARBS_TILE_SIZE), fy0 = floor((my - rd) / DARBS_TILE_SIZE);
    double fx1 = floor((mx + rd) / DARBS_TILE_SIZE), fy1 = floor((my + rd) / DARBS_TILE_SIZE);
    // NaN centres compare false everywhere -> empty rect, like an
    // int-converted NaN would be garbage in the reference (unsupported).
    if (fx1 >= 0.0 && fy1 >= 0.0 && fx0 <= tiles_x - 1 && fy0 <= tiles_y - 1) {
        int x0 = (int)fmax(fx0, 0.0), y0 = (int)fmax(fy0, 0.0);
        int x1 = (int)fmin(fx1, (double)(tiles_x - 1)), y1 = (int)fmin(fy1, (double)(tiles_y - 1));
        if (x1 >= x0 && y1 >= y0) {
            cnt = (unsigned)(x1 - x0 + 1) * (unsigned)(y1 - y0 + 1);
            rect = make_uint2((unsigned)x0 | ((unsigned)y0 << 16), (unsigned)x1 | ((unsigned)y1 << 16));
        }
    }
}

// K = the total of the tile counts: one atomic per warp, spread over kSlotsK addresses so that
// the ~8 k warps of a million splats do not serialise on one.  Every thread of the (possibly
// partial) warp that is still running calls this.
__device__ __forceinline__ void accumulate_tile_count(unsigned cnt, unsigned long long* k_slots) {
    const unsigned active = __activemask();
    const unsigned sum = __reduce_add_sync(active, cnt);
    if ((threadIdx.x & 31) == __ffs(active) - 1 && sum)
        atomicAdd(k_slots + (blockIdx.x & (kSlotsK - 1)), (unsigned long long)sum);
}

constexpr double kMaxKappa = 50.0;  // largest eigenvalue ratio of a conic the float32 decisions are trusted with

__device__ __forceinline__ void splat_record(const KParams& kp, float mx, float my, float a, float b, float c,
                                             float o, float cr, float cg, float cb, float4* __restrict__ r) {
    double ad = a, bd = b, cd = c;
    double thr = family_threshold(kp, (double)o);
    // An indefinite or non-finite conic cannot be culled by the convex block
    // test and may produce dm2 < 0 (rasterizer.cpp:91): force the FP64 path.
    bool pd = (ad > 0.0) && (cd > 0.0) && (ad * cd - bd * bd > 0.0);
    // The float32 quadratic form A dx^2 + B dx dy + C dy^2 is evaluated in absolute pixel offsets:
    // its terms reach kappa * m (kappa = the conic's eigenvalue ratio) and cancel down to m, so its
    // error is ~3 eps kappa m.  Past kappa = kMaxKappa that leaves the guard band (1e-4 at m ~ 10):
    // such needles (sigma 100 px against the 0.3 px^2 dilation floor) take every decision in FP64.
    if (pd) {
        const double tr = ad + cd, disc = sqrt((ad - cd) * (ad - cd) + 4.0 * bd * bd);
        pd = (tr + disc) <= kMaxKappa * (tr - disc);
    }
    float thr_m = pd ? (float)(thr * (double)kp.scale) : __int_as_float(0x7fc00000);
    // (A, C) adjacent: they meet (dx, dy) in one packed multiply (quad_m, render.cu)
    r[0] = make_float4(mx, my, kp.scale * a, kp.scale * c);
    // cull helpers: minimiser slope along the other axis, -B/(2C) and -B/(2A)
    r[1] = make_float4(kp.scale * (2.0f * b), o, thr_m, -b / c);
    r[2] = make_float4(cr, cg, cb, -b / a);
    r[3] = make_float4(a, b, c, 0.f);
}

}  // namespace darbs_b200
