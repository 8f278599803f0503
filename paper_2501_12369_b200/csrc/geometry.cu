// geometry.cu — per-primitive preprocess and its reverse, the reparametrisation
// chain of the training step, Adam and the L1 loss.
//
// Reference: realize                 src/fit3d.cpp:17-25
//            project_primitive       src/geometry.cpp:66-87 (+ :9-64)
//            backward_projection     src/geometry.cpp:111-168
//            conic-grad -> cov2-grad src/fit3d.cpp:140-144
//            reparametrisation, +=   src/fit3d.cpp:148-158
//            adam_step               include/darbs/optim.hpp:24-39
//            L1 part of loss_total   src/loss.cpp:183-188
//
// These stages stream ~100 B per primitive and do a few hundred flops on it:
// they are HBM-bound by a wide margin, so the arithmetic runs in FP64 on the
// float32 parameters (the B200 FP64 pipe is far from the limiter) and only the
// stored results are rounded to float32.  That keeps the integer-valued radius
// (ceil, geometry.cpp:62) and the near-plane test on the values the FP64
// reference sees.
#include "splat.cuh"

namespace darbs_b200 {

CameraD make_camera(const double* c) {
    CameraD cam;
    cam.fx = c[0];
    cam.fy = c[1];
    cam.cx = c[2];
    cam.cy = c[3];
    cam.width = (int)c[4];
    cam.height = (int)c[5];
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 4; ++k) cam.w[4 * r + k] = c[6 + 4 * r + k];
    return cam;
}

namespace {

enum { FLAG_INVALID = 1, FLAG_DEGENERATE = 2 };

// The per-primitive chain is written once, on a scalar type T: double where an integer is
// decided downstream (radius ceil, near plane, tile rectangle: project_kernel) or where the ABI
// promises the FP64 chain (backward_projection), float in the training step's gradient chain.
template <typename T>
__device__ __forceinline__ T sigmoid_out(float x);
template <>
__device__ __forceinline__ double sigmoid_out<double>(float x) { return (double)(1.0f / (1.0f + expf(-x))); }
template <>
__device__ __forceinline__ float sigmoid_out<float>(float x) { return 1.0f / (1.0f + __expf(-x)); }
template <typename T>
__device__ __forceinline__ T sigmoid_opacity(float x);
template <>
__device__ __forceinline__ double sigmoid_opacity<double>(float x) { return 1.0 / (1.0 + exp(-(double)x)); }
template <>
__device__ __forceinline__ float sigmoid_opacity<float>(float x) { return sigmoid_out<float>(x); }
__device__ __forceinline__ double exp_t(double x) { return exp(x); }
__device__ __forceinline__ float exp_t(float x) { return __expf(x); }
__device__ __forceinline__ double sqrt_t(double x) { return sqrt(x); }
__device__ __forceinline__ float sqrt_t(float x) { return sqrtf(x); }

template <typename T>
struct CameraT {
    T fx, fy, cx, cy;
    T w[12];  // rows 0..2 of the world-to-camera transform (3x4)
    __device__ explicit CameraT(const CameraD& c) : fx((T)c.fx), fy((T)c.fy), cx((T)c.cx), cy((T)c.cy) {
        for (int i = 0; i < 12; ++i) w[i] = (T)c.w[i];
    }
};

template <typename T>
struct PrimT {
    T mu[3], s[3], q[4], o, col[3];
};
using Prim = PrimT<double>;

template <typename T>
__device__ __forceinline__ void load_prim(const float* __restrict__ p, bool raw, PrimT<T>& out) {
    float v[14];
#pragma unroll
    for (int k = 0; k < 7; ++k) {
        float2 t = __ldg(reinterpret_cast<const float2*>(p) + k);
        v[2 * k] = t.x;
        v[2 * k + 1] = t.y;
    }
    for (int k = 0; k < 3; ++k) out.mu[k] = (T)v[k];
    for (int k = 0; k < 3; ++k) out.s[k] = raw ? exp_t((T)v[3 + k]) : (T)v[3 + k];
    for (int k = 0; k < 4; ++k) out.q[k] = (T)v[6 + k];
    // Colour leaves this chain as float32 and decides nothing: its sigmoids run in FP32 with the
    // accurate expf and division (<= 3 ulp), three of the chain's four FP64 exponentials otherwise.
    // Opacity DOES decide (alpha >= 1/255, the 0.99 clamp gate, and through alpha the entry at which
    // a pixel's transmittance crosses the floor): it is the reference's double sigmoid rounded once,
    // so the rasterizer sees the float32 value the reference's realisation rounds to.  (tests/
    // fuzz_cases.py: with an FP32 sigmoid, one ulp of opacity flipped a gate in 1 of ~200 views.)
    // (The float chain of the training step's gradients keeps the MUFU form: o (1 - o) only.)
    out.o = raw ? sigmoid_opacity<T>(v[10]) : (T)v[10];
    for (int k = 0; k < 3; ++k) out.col[k] = raw ? sigmoid_out<T>(v[11 + k]) : (T)v[11 + k];
}

// Quaternion (w,x,y,z) -> rotation matrix of its normalisation (Eigen's
// toRotationMatrix, used at geometry.cpp:13 and :115-116).
template <typename T>
__device__ __forceinline__ void quat_rot(const T* q, T* r, T* qn) {
    const T one = (T)1, two = (T)2;
    T n = sqrt_t(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    T w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
    qn[0] = w;
    qn[1] = x;
    qn[2] = y;
    qn[3] = z;
    T tx = two * x, ty = two * y, tz = two * z;
    T twx = tx * w, twy = ty * w, twz = tz * w;
    T txx = tx * x, txy = ty * x, txz = tz * x;
    T tyy = ty * y, tyz = tz * y, tzz = tz * z;
    r[0] = one - (tyy + tzz);
    r[1] = txy - twz;
    r[2] = txz + twy;
    r[3] = txy + twz;
    r[4] = one - (txx + tzz);
    r[5] = tyz - twx;
    r[6] = txz - twy;
    r[7] = tyz + twx;
    r[8] = one - (txx + tyy);
}

template <typename T>
struct ProjectedT {
    T t[3];     // camera-space mean
    T r[9];     // rotation of the primitive
    T qn[4];
    T tj[6];    // J * W_rot
    T sigma[9];
    T cov[3];   // xx, xy, yy after psi and dilation
};
using Projected = ProjectedT<double>;

// project_point / covariance_from_scale_rot / project_covariance / apply_psi
template <typename T>
__device__ __forceinline__ bool project_core(const PrimT<T>& p, const CameraT<T>& cam, T psi, T dilation,
                                             ProjectedT<T>& out) {
    const T half = (T)0.5;
    for (int r = 0; r < 3; ++r)
        out.t[r] = cam.w[4 * r] * p.mu[0] + cam.w[4 * r + 1] * p.mu[1] + cam.w[4 * r + 2] * p.mu[2] +
                   cam.w[4 * r + 3];
    if (out.t[2] <= (T)DARBS_NEAR_PLANE) return false;  // geometry.cpp:22
    quat_rot(p.q, out.r, out.qn);
    // Sigma = R diag(s^2) R^T, symmetrised (geometry.cpp:13-16)
    T rd[9];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) rd[3 * a + b] = out.r[3 * a + b] * (p.s[b] * p.s[b]);
    T m[9];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            m[3 * a + b] = rd[3 * a] * out.r[3 * b] + rd[3 * a + 1] * out.r[3 * b + 1] +
                           rd[3 * a + 2] * out.r[3 * b + 2];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) out.sigma[3 * a + b] = half * (m[3 * a + b] + m[3 * b + a]);
    // J (geometry.cpp:29-35) and T = J W_rot (:38)
    T z = out.t[2];
    T j[6] = {cam.fx / z, (T)0, -cam.fx * out.t[0] / (z * z), (T)0, cam.fy / z, -cam.fy * out.t[1] / (z * z)};
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b)
            out.tj[3 * a + b] = j[3 * a] * cam.w[b] + j[3 * a + 1] * cam.w[4 + b] + j[3 * a + 2] * cam.w[8 + b];
    T ts[6];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b)
            ts[3 * a + b] = out.tj[3 * a] * out.sigma[b] + out.tj[3 * a + 1] * out.sigma[3 + b] +
                            out.tj[3 * a + 2] * out.sigma[6 + b];
    T raw[4];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
            raw[2 * a + b] = ts[3 * a] * out.tj[3 * b] + ts[3 * a + 1] * out.tj[3 * b + 1] +
                             ts[3 * a + 2] * out.tj[3 * b + 2];
    T rxy = half * (raw[1] + raw[2]);
    out.cov[0] = psi * raw[0] + dilation;  // geometry.cpp:47
    out.cov[1] = psi * rxy;
    out.cov[2] = psi * raw[3] + dilation;
    return true;
}

__global__ void realize_kernel(int64_t n, const float* __restrict__ raw, float* __restrict__ prims) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    Prim p;
    load_prim(raw + 14 * i, true, p);
    float* o = prims + 14 * i;
    for (int k = 0; k < 3; ++k) o[k] = (float)p.mu[k];
    for (int k = 0; k < 3; ++k) o[3 + k] = (float)p.s[k];
    for (int k = 0; k < 4; ++k) o[6 + k] = (float)p.q[k];
    o[10] = (float)p.o;
    for (int k = 0; k < 3; ++k) o[11 + k] = (float)p.col[k];
}

__global__ void project_kernel(KParams kp, double psi, double dilation, int64_t n,
                               const float* __restrict__ params, bool raw, CameraD cam_d,
                               int* __restrict__ valid, float* __restrict__ mu2,
                               float* __restrict__ cov2, float* __restrict__ conic,
                               float* __restrict__ radius, float* __restrict__ depth,
                               float* __restrict__ opacity, float* __restrict__ rgb,
                               int* __restrict__ flags, SplatSinks sinks) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool in = i < n;
    const CameraT<double> cam(cam_d);
    Prim p;
    Projected pr;
    bool vis = false;
    if (in) {
        load_prim(params + 14 * i, raw, p);
        vis = project_core(p, cam, psi, dilation, pr);
    }
    float o_mu[2] = {0.f, 0.f}, o_cov[3] = {0.f, 0.f, 0.f}, o_con[3] = {0.f, 0.f, 0.f};
    float o_rad = 0.f, o_dep = 0.f;
    if (vis) {
        if (!(fmin(p.s[0], fmin(p.s[1], p.s[2])) > 0.0)) atomicOr(flags, FLAG_INVALID);  // geometry.cpp:10-12
        double a = pr.cov[0], b = pr.cov[1], c = pr.cov[2];
        double det = a * c - b * b;
        if (!(det > 0.0) || !(a > 0.0)) {  // geometry.cpp:53-55
            atomicOr(flags, FLAG_DEGENERATE);
            vis = false;
        } else {
            double mid = 0.5 * (a + c);
            double disc = sqrt(fmax(0.0, mid * mid - det));
            double l1 = mid + disc;
            o_con[0] = (float)(c / det);
            o_con[1] = (float)(-b / det);
            o_con[2] = (float)(a / det);
            o_rad = (float)ceil(sqrt(kp.cutoff_d) * sqrt(l1));  // geometry.cpp:62
            o_mu[0] = (float)(cam.fx * pr.t[0] / pr.t[2] + cam.cx);
            o_mu[1] = (float)(cam.fy * pr.t[1] / pr.t[2] + cam.cy);
            o_dep = (float)pr.t[2];
            o_cov[0] = (float)a;
            o_cov[1] = (float)b;
            o_cov[2] = (float)c;
        }
    }
    // visible-primitive count for the "all primitives culled" check (fit3d.cpp:117-119)
    unsigned bal = __ballot_sync(0xffffffffu, vis);
    if ((threadIdx.x & 31) == 0 && bal) atomicAdd(flags + 1, __popc(bal));
    if (!in) return;
    if (valid) valid[i] = vis ? 1 : 0;
    mu2[2 * i] = o_mu[0];
    mu2[2 * i + 1] = o_mu[1];
    if (cov2) {
        cov2[3 * i] = o_cov[0];
        cov2[3 * i + 1] = o_cov[1];
        cov2[3 * i + 2] = o_cov[2];
    }
    conic[3 * i] = o_con[0];
    conic[3 * i + 1] = o_con[1];
    conic[3 * i + 2] = o_con[2];
    radius[i] = o_rad;
    depth[i] = o_dep;
    if (opacity) opacity[i] = (float)p.o;
    if (rgb) {
        rgb[3 * i] = (float)p.col[0];
        rgb[3 * i + 1] = (float)p.col[1];
        rgb[3 * i + 2] = (float)p.col[2];
    }
    // training step: what rect_kernel and pack_kernel would derive from the arrays just written
    // (same float32 values in, same bits out), without a second and third pass over them
    if (sinks.recs) {
        uint2 rect;
        unsigned cnt;
        splat_rect(vis, o_mu[0], o_mu[1], o_con[0], o_con[1], o_con[2], o_rad, sinks.tiles_x, sinks.tiles_y,
                   sinks.skipped_nonfinite, rect, cnt);
        sinks.rects[i] = rect;
        sinks.touched[i] = cnt;
        accumulate_tile_count(cnt, sinks.k_slots);
        sinks.depth_keys[i] = depth_to_key(o_dep);
        sinks.order[i] = (unsigned)i;
        splat_record(kp, o_mu[0], o_mu[1], o_con[0], o_con[1], o_con[2], (float)p.o, (float)p.col[0],
                     (float)p.col[1], (float)p.col[2], sinks.recs + kRecVecs * i);
    }
}

// dR/dq of the unit-quaternion rotation, geometry.cpp:92-107 (already x2).
template <typename T>
__device__ __forceinline__ void rotation_jacobians(const T* q, T dr[4][9]) {
    const T two = (T)2, o = (T)0;
    T w = q[0], x = q[1], y = q[2], z = q[3];
    T d0[9] = {o, -z, y, z, o, -x, -y, x, o};
    T d1[9] = {o, y, z, y, -two * x, -w, z, w, -two * x};
    T d2[9] = {-two * y, x, w, x, o, z, -w, z, -two * y};
    T d3[9] = {-two * z, -w, x, w, -two * z, y, x, y, o};
    for (int i = 0; i < 9; ++i) {
        dr[0][i] = two * d0[i];
        dr[1][i] = two * d1[i];
        dr[2][i] = two * d2[i];
        dr[3][i] = two * d3[i];
    }
}

// backward_projection geometry.cpp:111-168.  gcov = (xx, xy, yx, yy).
template <typename T>
__device__ __forceinline__ void backward_projection_core(const PrimT<T>& p, const CameraT<T>& cam,
                                                         const ProjectedT<T>& pr, T psi, const T* gcov,
                                                         const T* gmu2, T* d_mu, T* d_scale, T* d_rot) {
    const T half = (T)0.5, two = (T)2;
    // sqrt factor M = R diag(s), Sigma = M M^T (:117-118)
    T m[9], sigma[9];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) m[3 * a + b] = pr.r[3 * a + b] * p.s[b];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            sigma[3 * a + b] = m[3 * a] * m[3 * b] + m[3 * a + 1] * m[3 * b + 1] + m[3 * a + 2] * m[3 * b + 2];
    const T* tj = pr.tj;
    const T* t = pr.t;
    T z = t[2];
    T gxy = half * (gcov[1] + gcov[2]);
    T graw[4] = {psi * gcov[0], psi * gxy, psi * gxy, psi * gcov[3]};  // :128-129
    T gt[6];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b) gt[3 * a + b] = graw[2 * a] * tj[b] + graw[2 * a + 1] * tj[3 + b];
    T d_sigma[9];  // :130
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) d_sigma[3 * a + b] = tj[a] * gt[b] + tj[3 + a] * gt[3 + b];
    T d_tj[6], d_j[6];  // :131-132
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b)
            d_tj[3 * a + b] = two * (gt[3 * a] * sigma[b] + gt[3 * a + 1] * sigma[3 + b] + gt[3 * a + 2] * sigma[6 + b]);
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b)
            d_j[3 * a + b] = d_tj[3 * a] * cam.w[4 * b] + d_tj[3 * a + 1] * cam.w[4 * b + 1] +
                             d_tj[3 * a + 2] * cam.w[4 * b + 2];
    T d_t[3];  // :135-145
    T z2 = z * z, z3 = z2 * z;
    d_t[0] = d_j[2] * (-cam.fx / z2);
    d_t[1] = d_j[5] * (-cam.fy / z2);
    d_t[2] = d_j[0] * (-cam.fx / z2) + d_j[4] * (-cam.fy / z2) + d_j[2] * (two * cam.fx * t[0] / z3) +
             d_j[5] * (two * cam.fy * t[1] / z3);
    d_t[0] += gmu2[0] * cam.fx / z;
    d_t[1] += gmu2[1] * cam.fy / z;
    d_t[2] += -gmu2[0] * cam.fx * t[0] / z2 - gmu2[1] * cam.fy * t[1] / z2;
    for (int a = 0; a < 3; ++a)  // :147
        d_mu[a] = cam.w[a] * d_t[0] + cam.w[4 + a] * d_t[1] + cam.w[8 + a] * d_t[2];
    T d_m[9], d_r[9];  // :150-152
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
            T acc = (T)0;
            for (int c = 0; c < 3; ++c) acc += (d_sigma[3 * a + c] + d_sigma[3 * c + a]) * m[3 * c + b];
            d_m[3 * a + b] = acc;
        }
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) d_r[3 * a + b] = d_m[3 * a + b] * p.s[b];
    for (int a = 0; a < 3; ++a)
        d_scale[a] = pr.r[a] * d_m[a] + pr.r[3 + a] * d_m[3 + a] + pr.r[6 + a] * d_m[6 + a];
    T dr[4][9], d_qn[4];  // :154-160
    rotation_jacobians(pr.qn, dr);
    for (int i = 0; i < 4; ++i) {
        T acc = (T)0;
        for (int e = 0; e < 9; ++e) acc += d_r[e] * dr[i][e];
        d_qn[i] = acc;
    }
    T norm = sqrt_t(p.q[0] * p.q[0] + p.q[1] * p.q[1] + p.q[2] * p.q[2] + p.q[3] * p.q[3]);  // :163-166
    T qu[4], dot = (T)0;
    for (int i = 0; i < 4; ++i) qu[i] = p.q[i] / norm;
    for (int i = 0; i < 4; ++i) dot += qu[i] * d_qn[i];
    for (int i = 0; i < 4; ++i) d_rot[i] = (d_qn[i] - qu[i] * dot) / norm;
}

__global__ void backward_projection_kernel(double psi, int64_t n, const float* __restrict__ grad_cov2,
                                           const float* __restrict__ grad_mu2,
                                           const float* __restrict__ prims, CameraD cam_d,
                                           float* __restrict__ d_mu, float* __restrict__ d_scale,
                                           float* __restrict__ d_rot) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const CameraT<double> cam(cam_d);
    Prim p;
    load_prim(prims + 14 * i, false, p);
    Projected pr;
    // The reference's backward_projection has no cull; evaluate the same
    // expressions whatever the depth (dilation does not enter the gradient).
    project_core(p, cam, psi, 0.0, pr);
    if (pr.t[2] <= DARBS_NEAR_PLANE) {
        // project_core returned before filling r/tj: fill them (rare path).
        quat_rot(p.q, pr.r, pr.qn);
        double z = pr.t[2];
        double j[6] = {cam.fx / z, 0.0, -cam.fx * pr.t[0] / (z * z), 0.0, cam.fy / z, -cam.fy * pr.t[1] / (z * z)};
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 3; ++b)
                pr.tj[3 * a + b] = j[3 * a] * cam.w[b] + j[3 * a + 1] * cam.w[4 + b] + j[3 * a + 2] * cam.w[8 + b];
    }
    double gc[4] = {grad_cov2[4 * i], grad_cov2[4 * i + 1], grad_cov2[4 * i + 2], grad_cov2[4 * i + 3]};
    double gm[2] = {grad_mu2[2 * i], grad_mu2[2 * i + 1]};
    double dm[3], ds[3], dq[4];
    backward_projection_core(p, cam, pr, psi, gc, gm, dm, ds, dq);
    for (int a = 0; a < 3; ++a) d_mu[3 * i + a] = (float)dm[a];
    for (int a = 0; a < 3; ++a) d_scale[3 * i + a] = (float)ds[a];
    for (int a = 0; a < 4; ++a) d_rot[4 * i + a] = (float)dq[a];
}

// fit3d.cpp:134-159 for one view, one thread per primitive (no compaction: a
// culled primitive has valid == 0 and simply adds nothing).  The whole chain in
// FP32: nothing here decides an integer, and the parity bar on parameter gradients
// (1e-3 relative) leaves four digits of head-room over float32 round-off.
// 64 registers (a few spilled words) for 8 CTAs per SM: the kernel waits on its loads, and the
// extra resident warps are worth more than the spills (70 -> 56 us at 1 M primitives)
__global__ void __launch_bounds__(128, 8)
param_grads_kernel(double psi_d, int64_t n, const float* __restrict__ raw, CameraD cam_d,
                   const int* __restrict__ valid, const float* __restrict__ splat_grads,
                   float* __restrict__ param_grads, bool overwrite) {
    using T = float;
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    float2* g = reinterpret_cast<float2*>(param_grads + 14 * i);
    if (!valid[i]) {  // culled in this view: adds nothing (and is cleared when this view overwrites)
        if (overwrite)
            for (int k = 0; k < 7; ++k) g[k] = make_float2(0.f, 0.f);
        return;
    }
    const CameraT<T> cam(cam_d);
    const T psi = (T)psi_d;
    PrimT<T> p;
    load_prim(raw + 14 * i, true, p);
    ProjectedT<T> pr;
    if (!project_core(p, cam, psi, (T)DARBS_DILATION, pr)) {
        if (overwrite)
            for (int k = 0; k < 7; ++k) g[k] = make_float2(0.f, 0.f);
        return;
    }
    // padded rows, SplatGrads order in the first nine
    const float4* gi4 = reinterpret_cast<const float4*>(splat_grads + kSplatGradRow * i);
    const float4 g0 = __ldg(gi4), g1 = __ldg(gi4 + 1);
    const float g8 = __ldg(splat_grads + kSplatGradRow * i + 8);
    T a = pr.cov[0], b = pr.cov[1], c = pr.cov[2];
    T inv = 1.0f / (a * c - b * b);
    T ca = c * inv, cb = -b * inv, cc = a * inv;  // conic, geometry.cpp:61
    // d_cov2 = -C G C with G = [[da, db/2],[db/2, dc]] (fit3d.cpp:140-144)
    T ga = g1.x, gb = 0.5f * g1.y, gc = g1.z;
    T t00 = -(ca * ga + cb * gb), t01 = -(ca * gb + cb * gc);
    T t10 = -(cb * ga + cc * gb), t11 = -(cb * gb + cc * gc);
    T dcov[4] = {t00 * ca + t01 * cb, t00 * cb + t01 * cc, t10 * ca + t11 * cb, t10 * cb + t11 * cc};
    T gm[2] = {g1.w, g8};
    T dm[3], ds[3], dq[4];
    backward_projection_core(p, cam, pr, psi, dcov, gm, dm, ds, dq);
    // fit3d.cpp:148-158: grads[owner] += ..., 14 floats per primitive as seven 64-bit read-modify-writes
    const float add[14] = {dm[0], dm[1], dm[2], ds[0] * p.s[0], ds[1] * p.s[1], ds[2] * p.s[2], dq[0], dq[1],
                           dq[2], dq[3], g0.w * p.o * (1.0f - p.o), g0.x * p.col[0] * (1.0f - p.col[0]),
                           g0.y * p.col[1] * (1.0f - p.col[1]), g0.z * p.col[2] * (1.0f - p.col[2])};
#pragma unroll
    for (int k = 0; k < 7; ++k) {
        float2 v = overwrite ? make_float2(0.f, 0.f) : g[k];
        v.x += add[2 * k];
        v.y += add[2 * k + 1];
        g[k] = v;
    }
}

// adam_step optim.hpp:24-39, four parameters per thread (the launcher peels the tail and falls
// back to scalars when an array is not 16-byte aligned).
__device__ __forceinline__ void adam_one(float& p, float g, float& m, float& v, float lr, float inv_bc1,
                                         float inv_bc2) {
    const float b1 = 0.9f, b2 = 0.999f, eps = 1e-15f;  // optim.hpp:19-21
    m = b1 * m + (1.0f - b1) * g;
    v = b2 * v + (1.0f - b2) * g * g;
    p -= lr * (m * inv_bc1) / (sqrtf(v * inv_bc2) + eps);
}

__global__ void adam_kernel(int64_t dim4, int64_t dim, float* __restrict__ params,
                            const float* __restrict__ grads, float* __restrict__ m,
                            float* __restrict__ v, const float* __restrict__ lrs, float inv_bc1,
                            float inv_bc2) {
    // Blocks walk the arrays from the end: the gradients param_grads_kernel wrote last are still in
    // L2, and the parameters this kernel writes last (the front of the array) are the ones the next
    // iteration's project_kernel reads first.
    const int64_t i = (gridDim.x - 1 - blockIdx.x) * (int64_t)blockDim.x + threadIdx.x;
    if (i < dim4) {
        float4 p = reinterpret_cast<float4*>(params)[i];
        const float4 g = __ldg(reinterpret_cast<const float4*>(grads) + i);
        float4 mm = reinterpret_cast<float4*>(m)[i], vv = reinterpret_cast<float4*>(v)[i];
        const float4 lr = __ldg(reinterpret_cast<const float4*>(lrs) + i);
        adam_one(p.x, g.x, mm.x, vv.x, lr.x, inv_bc1, inv_bc2);
        adam_one(p.y, g.y, mm.y, vv.y, lr.y, inv_bc1, inv_bc2);
        adam_one(p.z, g.z, mm.z, vv.z, lr.z, inv_bc1, inv_bc2);
        adam_one(p.w, g.w, mm.w, vv.w, lr.w, inv_bc1, inv_bc2);
        reinterpret_cast<float4*>(params)[i] = p;
        reinterpret_cast<float4*>(m)[i] = mm;
        reinterpret_cast<float4*>(v)[i] = vv;
    } else {
        const int64_t j = 4 * dim4 + (i - dim4);
        if (j < dim) adam_one(params[j], grads[j], m[j], v[j], lrs[j], inv_bc1, inv_bc2);
    }
}

// loss.cpp:183-188 with lambda == 0: grad = sign(d)/n; sums[0] += |d|, sums[1] += d^2.  One float4
// per thread per step, FP32 partial sums per thread (a few hundred terms), FP64 across threads.
__global__ void __launch_bounds__(256)
l1_loss_kernel(int64_t count4, int64_t count, const float* __restrict__ image,
               const float* __restrict__ target, float coef, float* __restrict__ grad,
               double* __restrict__ sums) {
    __shared__ double red[2][8];
    float s1 = 0.f, s2 = 0.f;
    auto one = [&](float a, float b) {
        const float d = a - b;
        s1 += fabsf(d);
        s2 = fmaf(d, d, s2);
        return coef * (float)((d > 0.f) - (d < 0.f));
    };
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count4;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(image) + i);
        const float4 b = __ldg(reinterpret_cast<const float4*>(target) + i);
        float4 r;
        r.x = one(a.x, b.x);
        r.y = one(a.y, b.y);
        r.z = one(a.z, b.z);
        r.w = one(a.w, b.w);
        reinterpret_cast<float4*>(grad)[i] = r;
    }
    if (blockIdx.x == 0)
        for (int64_t j = 4 * count4 + threadIdx.x; j < count; j += blockDim.x) grad[j] = one(image[j], target[j]);
    double d1 = s1, d2 = s2;
    for (int o = 16; o > 0; o >>= 1) {
        d1 += __shfl_xor_sync(0xffffffffu, d1, o);
        d2 += __shfl_xor_sync(0xffffffffu, d2, o);
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = d1;
        red[1][threadIdx.x >> 5] = d2;
    }
    __syncthreads();
    if (threadIdx.x < 2) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[threadIdx.x][w];
        atomicAdd(sums + threadIdx.x, t);
    }
}

inline unsigned grid_for(int64_t n, int threads) { return (unsigned)((n + threads - 1) / threads); }

}  // namespace

darbs_status launch_realize(darbs_cuda_ctx* ctx, int64_t n, const float* raw, float* prims) {
    if (n == 0) return DARBS_OK;
    realize_kernel<<<grid_for(n, 128), 128, 0, ctx->stream>>>(n, raw, prims);
    return check_launch(ctx, "realize_kernel");
}

darbs_status launch_project(darbs_cuda_ctx* ctx, const KParams& kp, double psi, double dilation,
                            int64_t n, const float* params, bool raw, const CameraD& cam,
                            int32_t* valid, float* mu2, float* cov2, float* conic, float* radius,
                            float* depth, float* opacity, float* rgb, int* status_flags,
                            const SplatSinks* sinks) {
    if (n == 0) return DARBS_OK;
    project_kernel<<<grid_for(n, 128), 128, 0, ctx->stream>>>(kp, psi, dilation, n, params, raw, cam,
                                                             valid, mu2, cov2, conic, radius, depth,
                                                             opacity, rgb, status_flags,
                                                             sinks ? *sinks : SplatSinks());
    return check_launch(ctx, "project_kernel");
}

darbs_status launch_backward_projection(darbs_cuda_ctx* ctx, double psi, int64_t n,
                                        const float* grad_cov2, const float* grad_mu2,
                                        const float* prims, const CameraD& cam, float* d_mu,
                                        float* d_scale, float* d_rot) {
    if (n == 0) return DARBS_OK;
    backward_projection_kernel<<<grid_for(n, 128), 128, 0, ctx->stream>>>(
        psi, n, grad_cov2, grad_mu2, prims, cam, d_mu, d_scale, d_rot);
    return check_launch(ctx, "backward_projection_kernel");
}

darbs_status launch_param_grads(darbs_cuda_ctx* ctx, double psi, int64_t n, const float* raw,
                                const CameraD& cam, const int32_t* valid, const float* splat_grads,
                                const float* /*conic*/, float* param_grads, bool overwrite) {
    if (n == 0) return DARBS_OK;
    param_grads_kernel<<<grid_for(n, 128), 128, 0, ctx->stream>>>(psi, n, raw, cam, valid, splat_grads,
                                                                 param_grads, overwrite);
    return check_launch(ctx, "param_grads_kernel");
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

darbs_status launch_adam(darbs_cuda_ctx* ctx, int64_t dim, float* params, const float* grads,
                         float* m, float* v, const float* lrs, int t) {
    if (dim == 0) return DARBS_OK;
    double bc1 = 1.0 - pow(0.9, t), bc2 = 1.0 - pow(0.999, t);
    const bool vec = aligned16(params) && aligned16(grads) && aligned16(m) && aligned16(v) && aligned16(lrs);
    const int64_t dim4 = vec ? dim / 4 : 0;
    const int64_t threads = dim4 + (dim - 4 * dim4);
    adam_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, ctx->stream>>>(
        dim4, dim, params, grads, m, v, lrs, (float)(1.0 / bc1), (float)(1.0 / bc2));
    return check_launch(ctx, "adam_kernel");
}

darbs_status launch_l1_loss(darbs_cuda_ctx* ctx, int64_t count, const float* image,
                            const float* target, double lambda, float* grad_image,
                            double* sums) {
    DARBS_CUDA_TRY(ctx, cudaMemsetAsync(sums, 0, sizeof(double) * 2, ctx->stream));
    if (count == 0) return DARBS_OK;
    float coef = (float)((1.0 - lambda) / (double)count);
    const bool vec = aligned16(image) && aligned16(target) && aligned16(grad_image);
    l1_loss_kernel<<<148 * 8, 256, 0, ctx->stream>>>(vec ? count / 4 : 0, count, image, target, coef, grad_image,
                                                     sums);
    return check_launch(ctx, "l1_loss_kernel");
}

}  // namespace darbs_b200
