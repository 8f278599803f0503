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
#include "family.cuh"

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

struct Prim {
    double mu[3], s[3], q[4], o, col[3];
};

__device__ __forceinline__ double sigmoid_d(double x) { return 1.0 / (1.0 + exp(-x)); }

__device__ __forceinline__ void load_prim(const float* __restrict__ p, bool raw, Prim& out) {
    float v[14];
#pragma unroll
    for (int k = 0; k < 7; ++k) {
        float2 t = __ldg(reinterpret_cast<const float2*>(p) + k);
        v[2 * k] = t.x;
        v[2 * k + 1] = t.y;
    }
    for (int k = 0; k < 3; ++k) out.mu[k] = v[k];
    for (int k = 0; k < 3; ++k) out.s[k] = raw ? exp((double)v[3 + k]) : (double)v[3 + k];
    for (int k = 0; k < 4; ++k) out.q[k] = v[6 + k];
    out.o = raw ? sigmoid_d(v[10]) : (double)v[10];
    for (int k = 0; k < 3; ++k) out.col[k] = raw ? sigmoid_d(v[11 + k]) : (double)v[11 + k];
}

// Quaternion (w,x,y,z) -> rotation matrix of its normalisation (Eigen's
// toRotationMatrix, used at geometry.cpp:13 and :115-116).
__device__ __forceinline__ void quat_rot(const double* q, double* r, double* qn) {
    double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    double w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
    qn[0] = w;
    qn[1] = x;
    qn[2] = y;
    qn[3] = z;
    double tx = 2.0 * x, ty = 2.0 * y, tz = 2.0 * z;
    double twx = tx * w, twy = ty * w, twz = tz * w;
    double txx = tx * x, txy = ty * x, txz = tz * x;
    double tyy = ty * y, tyz = tz * y, tzz = tz * z;
    r[0] = 1.0 - (tyy + tzz);
    r[1] = txy - twz;
    r[2] = txz + twy;
    r[3] = txy + twz;
    r[4] = 1.0 - (txx + tzz);
    r[5] = tyz - twx;
    r[6] = txz - twy;
    r[7] = tyz + twx;
    r[8] = 1.0 - (txx + tyy);
}

struct Projected {
    double t[3];     // camera-space mean
    double r[9];     // rotation of the primitive
    double qn[4];
    double tj[6];    // J * W_rot
    double sigma[9];
    double cov[3];   // xx, xy, yy after psi and dilation
};

// project_point / covariance_from_scale_rot / project_covariance / apply_psi
__device__ __forceinline__ bool project_core(const Prim& p, const CameraD& cam, double psi,
                                             double dilation, Projected& out) {
    for (int r = 0; r < 3; ++r)
        out.t[r] = cam.w[4 * r] * p.mu[0] + cam.w[4 * r + 1] * p.mu[1] + cam.w[4 * r + 2] * p.mu[2] +
                   cam.w[4 * r + 3];
    if (out.t[2] <= DARBS_NEAR_PLANE) return false;  // geometry.cpp:22
    quat_rot(p.q, out.r, out.qn);
    // Sigma = R diag(s^2) R^T, symmetrised (geometry.cpp:13-16)
    double rd[9];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) rd[3 * a + b] = out.r[3 * a + b] * (p.s[b] * p.s[b]);
    double m[9];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            m[3 * a + b] = rd[3 * a] * out.r[3 * b] + rd[3 * a + 1] * out.r[3 * b + 1] +
                           rd[3 * a + 2] * out.r[3 * b + 2];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) out.sigma[3 * a + b] = 0.5 * (m[3 * a + b] + m[3 * b + a]);
    // J (geometry.cpp:29-35) and T = J W_rot (:38)
    double z = out.t[2];
    double j[6] = {cam.fx / z, 0.0, -cam.fx * out.t[0] / (z * z),
                   0.0, cam.fy / z, -cam.fy * out.t[1] / (z * z)};
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b)
            out.tj[3 * a + b] = j[3 * a] * cam.w[b] + j[3 * a + 1] * cam.w[4 + b] + j[3 * a + 2] * cam.w[8 + b];
    double ts[6];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b)
            ts[3 * a + b] = out.tj[3 * a] * out.sigma[b] + out.tj[3 * a + 1] * out.sigma[3 + b] +
                            out.tj[3 * a + 2] * out.sigma[6 + b];
    double raw[4];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
            raw[2 * a + b] = ts[3 * a] * out.tj[3 * b] + ts[3 * a + 1] * out.tj[3 * b + 1] +
                             ts[3 * a + 2] * out.tj[3 * b + 2];
    double rxy = 0.5 * (raw[1] + raw[2]);
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
                               const float* __restrict__ params, bool raw, CameraD cam,
                               int* __restrict__ valid, float* __restrict__ mu2,
                               float* __restrict__ cov2, float* __restrict__ conic,
                               float* __restrict__ radius, float* __restrict__ depth,
                               float* __restrict__ opacity, float* __restrict__ rgb,
                               int* __restrict__ flags) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool in = i < n;
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
}

// dR/dq of the unit-quaternion rotation, geometry.cpp:92-107 (already x2).
__device__ __forceinline__ void rotation_jacobians(const double* q, double dr[4][9]) {
    double w = q[0], x = q[1], y = q[2], z = q[3];
    double d0[9] = {0, -z, y, z, 0, -x, -y, x, 0};
    double d1[9] = {0, y, z, y, -2 * x, -w, z, w, -2 * x};
    double d2[9] = {-2 * y, x, w, x, 0, z, -w, z, -2 * y};
    double d3[9] = {-2 * z, -w, x, w, -2 * z, y, x, y, 0};
    for (int i = 0; i < 9; ++i) {
        dr[0][i] = 2.0 * d0[i];
        dr[1][i] = 2.0 * d1[i];
        dr[2][i] = 2.0 * d2[i];
        dr[3][i] = 2.0 * d3[i];
    }
}

// backward_projection geometry.cpp:111-168.  gcov = (xx, xy, yx, yy).
__device__ __forceinline__ void backward_projection_core(const Prim& p, const CameraD& cam,
                                                         const Projected& pr, double psi,
                                                         const double* gcov, const double* gmu2,
                                                         double* d_mu, double* d_scale,
                                                         double* d_rot) {
    // sqrt factor M = R diag(s), Sigma = M M^T (:117-118)
    double m[9], sigma[9];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) m[3 * a + b] = pr.r[3 * a + b] * p.s[b];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            sigma[3 * a + b] = m[3 * a] * m[3 * b] + m[3 * a + 1] * m[3 * b + 1] + m[3 * a + 2] * m[3 * b + 2];
    const double* tj = pr.tj;
    const double* t = pr.t;
    double z = t[2];
    double gxy = 0.5 * (gcov[1] + gcov[2]);
    double graw[4] = {psi * gcov[0], psi * gxy, psi * gxy, psi * gcov[3]};  // :128-129
    double gt[6];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b) gt[3 * a + b] = graw[2 * a] * tj[b] + graw[2 * a + 1] * tj[3 + b];
    double d_sigma[9];  // :130
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) d_sigma[3 * a + b] = tj[a] * gt[b] + tj[3 + a] * gt[3 + b];
    double d_tj[6], d_j[6];  // :131-132
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b)
            d_tj[3 * a + b] = 2.0 * (gt[3 * a] * sigma[b] + gt[3 * a + 1] * sigma[3 + b] + gt[3 * a + 2] * sigma[6 + b]);
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b)
            d_j[3 * a + b] = d_tj[3 * a] * cam.w[4 * b] + d_tj[3 * a + 1] * cam.w[4 * b + 1] +
                             d_tj[3 * a + 2] * cam.w[4 * b + 2];
    double d_t[3];  // :135-145
    double z2 = z * z, z3 = z2 * z;
    d_t[0] = d_j[2] * (-cam.fx / z2);
    d_t[1] = d_j[5] * (-cam.fy / z2);
    d_t[2] = d_j[0] * (-cam.fx / z2) + d_j[4] * (-cam.fy / z2) + d_j[2] * (2.0 * cam.fx * t[0] / z3) +
             d_j[5] * (2.0 * cam.fy * t[1] / z3);
    d_t[0] += gmu2[0] * cam.fx / z;
    d_t[1] += gmu2[1] * cam.fy / z;
    d_t[2] += -gmu2[0] * cam.fx * t[0] / z2 - gmu2[1] * cam.fy * t[1] / z2;
    for (int a = 0; a < 3; ++a)  // :147
        d_mu[a] = cam.w[a] * d_t[0] + cam.w[4 + a] * d_t[1] + cam.w[8 + a] * d_t[2];
    double d_m[9], d_r[9];  // :150-152
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
            double acc = 0.0;
            for (int c = 0; c < 3; ++c) acc += (d_sigma[3 * a + c] + d_sigma[3 * c + a]) * m[3 * c + b];
            d_m[3 * a + b] = acc;
        }
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) d_r[3 * a + b] = d_m[3 * a + b] * p.s[b];
    for (int a = 0; a < 3; ++a)
        d_scale[a] = pr.r[a] * d_m[a] + pr.r[3 + a] * d_m[3 + a] + pr.r[6 + a] * d_m[6 + a];
    double dr[4][9], d_qn[4];  // :154-160
    rotation_jacobians(pr.qn, dr);
    for (int i = 0; i < 4; ++i) {
        double acc = 0.0;
        for (int e = 0; e < 9; ++e) acc += d_r[e] * dr[i][e];
        d_qn[i] = acc;
    }
    double norm = sqrt(p.q[0] * p.q[0] + p.q[1] * p.q[1] + p.q[2] * p.q[2] + p.q[3] * p.q[3]);  // :163-166
    double qu[4], dot = 0.0;
    for (int i = 0; i < 4; ++i) qu[i] = p.q[i] / norm;
    for (int i = 0; i < 4; ++i) dot += qu[i] * d_qn[i];
    for (int i = 0; i < 4; ++i) d_rot[i] = (d_qn[i] - qu[i] * dot) / norm;
}

__global__ void backward_projection_kernel(double psi, int64_t n, const float* __restrict__ grad_cov2,
                                           const float* __restrict__ grad_mu2,
                                           const float* __restrict__ prims, CameraD cam,
                                           float* __restrict__ d_mu, float* __restrict__ d_scale,
                                           float* __restrict__ d_rot) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
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
// culled primitive has valid == 0 and simply adds nothing).
__global__ void param_grads_kernel(double psi, int64_t n, const float* __restrict__ raw, CameraD cam,
                                   const int* __restrict__ valid,
                                   const float* __restrict__ splat_grads,
                                   float* __restrict__ param_grads) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (!valid[i]) return;
    Prim p;
    load_prim(raw + 14 * i, true, p);
    Projected pr;
    if (!project_core(p, cam, psi, DARBS_DILATION, pr)) return;
    const float* gi = splat_grads + kSplatGradRow * i;  // padded rows, SplatGrads order in the first nine
    double a = pr.cov[0], b = pr.cov[1], c = pr.cov[2];
    double det = a * c - b * b;
    double ca = c / det, cb = -b / det, cc = a / det;  // conic, geometry.cpp:61
    // d_cov2 = -C G C with G = [[da, db/2],[db/2, dc]] (fit3d.cpp:140-144)
    double ga = gi[4], gb = 0.5 * (double)gi[5], gc = gi[6];
    double t00 = -(ca * ga + cb * gb), t01 = -(ca * gb + cb * gc);
    double t10 = -(cb * ga + cc * gb), t11 = -(cb * gb + cc * gc);
    double dcov[4] = {t00 * ca + t01 * cb, t00 * cb + t01 * cc, t10 * ca + t11 * cb, t10 * cb + t11 * cc};
    double gm[2] = {gi[7], gi[8]};
    double dm[3], ds[3], dq[4];
    backward_projection_core(p, cam, pr, psi, dcov, gm, dm, ds, dq);
    float* g = param_grads + 14 * i;
    // fit3d.cpp:148-158
    g[0] += (float)dm[0];
    g[1] += (float)dm[1];
    g[2] += (float)dm[2];
    for (int k = 0; k < 3; ++k) g[3 + k] += (float)(ds[k] * p.s[k]);
    for (int k = 0; k < 4; ++k) g[6 + k] += (float)dq[k];
    g[10] += (float)((double)gi[3] * p.o * (1.0 - p.o));
    for (int k = 0; k < 3; ++k) g[11 + k] += (float)((double)gi[k] * p.col[k] * (1.0 - p.col[k]));
}

// adam_step optim.hpp:24-39
__global__ void adam_kernel(int64_t dim, float* __restrict__ params, const float* __restrict__ grads,
                            float* __restrict__ m, float* __restrict__ v,
                            const float* __restrict__ lrs, float inv_bc1, float inv_bc2) {
    const float b1 = 0.9f, b2 = 0.999f, eps = 1e-15f;  // optim.hpp:19-21
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < dim;
         i += (int64_t)gridDim.x * blockDim.x) {
        float g = grads[i];
        float mi = b1 * m[i] + (1.0f - b1) * g;
        float vi = b2 * v[i] + (1.0f - b2) * g * g;
        m[i] = mi;
        v[i] = vi;
        float mhat = mi * inv_bc1;
        float vhat = vi * inv_bc2;
        params[i] -= lrs[i] * mhat / (sqrtf(vhat) + eps);
    }
}

// loss.cpp:183-188 with lambda == 0: grad = sign(d)/n; sums[0] += |d|, sums[1] += d^2
__global__ void l1_loss_kernel(int64_t count, const float* __restrict__ image,
                               const float* __restrict__ target, float coef,
                               float* __restrict__ grad, double* __restrict__ sums) {
    double s1 = 0.0, s2 = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        float d = image[i] - target[i];
        s1 += fabsf(d);
        s2 += (double)d * d;
        grad[i] = coef * (float)((d > 0.f) - (d < 0.f));
    }
    for (int o = 16; o > 0; o >>= 1) {
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(sums, s1);
        atomicAdd(sums + 1, s2);
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
                            float* depth, float* opacity, float* rgb, int* status_flags) {
    if (n == 0) return DARBS_OK;
    project_kernel<<<grid_for(n, 128), 128, 0, ctx->stream>>>(kp, psi, dilation, n, params, raw, cam,
                                                             valid, mu2, cov2, conic, radius, depth,
                                                             opacity, rgb, status_flags);
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
                                const float* /*conic*/, float* param_grads) {
    if (n == 0) return DARBS_OK;
    param_grads_kernel<<<grid_for(n, 128), 128, 0, ctx->stream>>>(psi, n, raw, cam, valid, splat_grads,
                                                                 param_grads);
    return check_launch(ctx, "param_grads_kernel");
}

darbs_status launch_adam(darbs_cuda_ctx* ctx, int64_t dim, float* params, const float* grads,
                         float* m, float* v, const float* lrs, int t) {
    if (dim == 0) return DARBS_OK;
    double bc1 = 1.0 - pow(0.9, t), bc2 = 1.0 - pow(0.999, t);
    int64_t blocks = (dim + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    adam_kernel<<<(unsigned)blocks, 256, 0, ctx->stream>>>(dim, params, grads, m, v, lrs,
                                                          (float)(1.0 / bc1), (float)(1.0 / bc2));
    return check_launch(ctx, "adam_kernel");
}

darbs_status launch_l1_loss(darbs_cuda_ctx* ctx, int64_t count, const float* image,
                            const float* target, double lambda, float* grad_image,
                            double* sums) {
    DARBS_CUDA_TRY(ctx, cudaMemsetAsync(sums, 0, sizeof(double) * 2, ctx->stream));
    if (count == 0) return DARBS_OK;
    float coef = (float)((1.0 - lambda) / (double)count);
    l1_loss_kernel<<<148 * 8, 256, 0, ctx->stream>>>(count, image, target, coef, grad_image, sums);
    return check_launch(ctx, "l1_loss_kernel");
}

}  // namespace darbs_b200
