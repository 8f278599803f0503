/*
 * darbs_oracle.c — plain-C FP64 restatement of the reference's rasterizer hot
 * path ("port" oracle).
 *
 * TEST INFRASTRUCTURE, NOT PRODUCT: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load the library built
 * from this file, and only as the checker or the timed CPU baseline.
 *
 * Parity status: PINNED.  Every function below follows the reference lines it
 * cites (paths relative to /root/reference/proj/), and the result is checked
 *   (1) against the known-answer values of the reference's own unit tests
 *       (tests/test_kernel.cpp, tests/test_geometry.cpp,
 *       tests/test_rasterizer.cpp) re-expressed in tests/test_oracle_known_answers.py, and
 *   (2) against oracle/_ref/libdarbs_ref.so — the reference's own sources
 *       compiled unmodified (oracle/Makefile) — in tests/test_oracle_vs_ref.py and
 *       through the committed golden vectors under tests/golden/.
 * The only third-party dependency of the reference on this path is Eigen3
 * (>= 3.3, un-vendored, unpinned: core/CMakeLists.txt:1) for fixed-size 2x2 /
 * 3x3 / quaternion algebra; its published formulas (Quaternion::
 * toRotationMatrix, dense products) are written out longhand here.
 */
#define _GNU_SOURCE
#include "darbs_cpu.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define PI 3.14159265358979323846

const char* darbs_cpu_kind(void) { return "port"; }

/* ------------------------------------------------------------------ kernel */

/* is_bounded kernel.cpp:21-24 */
static int is_bounded(int f) {
    return f == DARBS_CPU_HALF_COSINE || f == DARBS_CPU_RAISED_COSINE ||
           f == DARBS_CPU_MODULUS_SINC;
}

/* u_limit kernel.cpp:27-38 */
static double u_limit(int family, int lobes) {
    switch (family) {
        case DARBS_CPU_HALF_COSINE:
            return PI / 2.0;
        case DARBS_CPU_RAISED_COSINE:
            return lobes * PI;
        case DARBS_CPU_MODULUS_SINC:
            return (lobes + 1) * PI / 2.0;
        default:
            return INFINITY;
    }
}

/* make_kernel kernel.cpp:42-65 */
int darbs_cpu_make_kernel(int family, double beta, double xi, int lobes, darbs_cpu_kernel* out) {
    if (!(beta > 0.0) || !isfinite(beta)) return DARBS_CPU_INVALID_PARAMETER;
    if (!(xi > 0.0) || !isfinite(xi)) return DARBS_CPU_INVALID_PARAMETER;
    if (lobes < 1) return DARBS_CPU_INVALID_PARAMETER;
    if (family < 0 || family > DARBS_CPU_INVERSE_MULTIQUADRATIC) return DARBS_CPU_INVALID_PARAMETER;
    out->family = family;
    out->beta = beta;
    out->xi = xi;
    out->lobes = lobes;
    out->unbounded = !is_bounded(family);
    if (out->unbounded) {
        out->cutoff = 3.0 * 3.0; /* kRenderCutoffDm kernel.cpp:19 */
    } else {
        out->cutoff = pow(xi * u_limit(family, lobes), 2.0 / beta);
    }
    return DARBS_CPU_OK;
}

/* kernel_preset kernel.cpp:223-240 */
int darbs_cpu_kernel_preset(const char* name, darbs_cpu_kernel* out) {
    if (!strcmp(name, "gaussian")) return darbs_cpu_make_kernel(DARBS_CPU_GAUSSIAN, 2.0, 2.0, 1, out);
    if (!strcmp(name, "half-cosine-sq"))
        return darbs_cpu_make_kernel(DARBS_CPU_HALF_COSINE, 2.0, 18.0 / PI, 1, out);
    if (!strcmp(name, "raised-cosine"))
        return darbs_cpu_make_kernel(DARBS_CPU_RAISED_COSINE, 1.0, 2.5 / PI, 1, out);
    if (!strcmp(name, "mod-sinc"))
        return darbs_cpu_make_kernel(DARBS_CPU_MODULUS_SINC, 1.0, 3.0 / PI, 1, out);
    if (!strcmp(name, "inv-multiquadratic"))
        return darbs_cpu_make_kernel(DARBS_CPU_INVERSE_MULTIQUADRATIC, 2.0, 1.0, 1, out);
    return DARBS_CPU_INVALID_PARAMETER;
}

/* kPsiDefaults psi_table.hpp:20-26 */
double darbs_cpu_default_psi(const char* name) {
    if (!strcmp(name, "gaussian")) return 1.0;
    if (!strcmp(name, "half-cosine-sq")) return 1.36;
    if (!strcmp(name, "raised-cosine")) return 0.6552;
    if (!strcmp(name, "mod-sinc")) return 1.1762;
    if (!strcmp(name, "inv-multiquadratic")) return 1.6054;
    return -1.0;
}

/* family_fu kernel.cpp:73-104 */
static void family_fu(int fam, double u, double* f, double* df) {
    switch (fam) {
        case DARBS_CPU_GAUSSIAN:
            *f = exp(-u);
            *df = -*f;
            return;
        case DARBS_CPU_HALF_COSINE:
            *f = cos(u);
            *df = -sin(u);
            return;
        case DARBS_CPU_RAISED_COSINE:
            *f = 0.5 + 0.5 * cos(u);
            *df = -0.5 * sin(u);
            return;
        case DARBS_CPU_MODULUS_SINC: {
            if (u < 1e-8) {
                *f = 1.0 - u * u / 6.0;
                *df = -u / 3.0;
                return;
            }
            double s = sin(u);
            double sgn = (double)((s > 0.0) - (s < 0.0));
            *f = fabs(s) / u;
            *df = sgn * (u * cos(u) - s) / (u * u);
            return;
        }
        default:
            *f = 0.0;
            *df = 0.0;
            return;
    }
}

/* center_dweight kernel.cpp:109-123 */
static double center_dweight(const darbs_cpu_kernel* s) {
    switch (s->family) {
        case DARBS_CPU_GAUSSIAN:
            return s->beta == 2.0 ? -1.0 / s->xi : 0.0;
        case DARBS_CPU_HALF_COSINE:
            return s->beta == 1.0 ? -1.0 / (2.0 * s->xi * s->xi) : 0.0;
        case DARBS_CPU_RAISED_COSINE:
            return s->beta == 1.0 ? -1.0 / (4.0 * s->xi * s->xi) : 0.0;
        case DARBS_CPU_MODULUS_SINC:
            return s->beta == 1.0 ? -1.0 / (6.0 * s->xi * s->xi) : 0.0;
        case DARBS_CPU_INVERSE_MULTIQUADRATIC:
            return -1.0 / (2.0 * s->xi);
    }
    return 0.0;
}

static inline double clamp01(double f) { return f < 0.0 ? 0.0 : (f > 1.0 ? 1.0 : f); }

/* eval kernel.cpp:127-164; the argument check (:128-130) is done by callers
 * that need the status (darbs_cpu_eval); the compositing loops only call this
 * with dm2 >= 0 (rasterizer.cpp:91). */
static inline void kernel_eval(const darbs_cpu_kernel* spec, double dm2, double* weight,
                               double* dweight) {
    *weight = 0.0;
    *dweight = 0.0;
    if (spec->unbounded ? dm2 > spec->cutoff : dm2 >= spec->cutoff) return;
    if (spec->family == DARBS_CPU_INVERSE_MULTIQUADRATIC) {
        double base = dm2 / spec->xi + 1.0;
        double r = 1.0 / sqrt(base);
        *weight = r;
        *dweight = -0.5 * r / (base * spec->xi);
        return;
    }
    if (dm2 < 1e-30) {
        double f, df;
        family_fu(spec->family, 0.0, &f, &df);
        *weight = f;
        *dweight = center_dweight(spec);
        return;
    }
    double u = (spec->beta == 2.0) ? dm2 / spec->xi : pow(dm2, 0.5 * spec->beta) / spec->xi;
    double f, df;
    family_fu(spec->family, u, &f, &df);
    double du = (spec->beta == 2.0)
                    ? 1.0 / spec->xi
                    : 0.5 * spec->beta * pow(dm2, 0.5 * spec->beta - 1.0) / spec->xi;
    *weight = clamp01(f);
    *dweight = df * du;
}

int darbs_cpu_eval(const darbs_cpu_kernel* k, int n, const double* dm2, double* weight,
                   double* dweight_ddm2) {
    for (int i = 0; i < n; ++i) {
        if (dm2[i] < 0.0 || !isfinite(dm2[i])) return DARBS_CPU_INVALID_PARAMETER; /* :128-130 */
        double w, dw;
        kernel_eval(k, dm2[i], &w, &dw);
        if (weight) weight[i] = w;
        if (dweight_ddm2) dweight_ddm2[i] = dw;
    }
    return DARBS_CPU_OK;
}

/* ---------------------------------------------------------------- geometry */

/* conic_and_radius geometry.cpp:50-64 */
static int conic_radius_one(const darbs_cpu_kernel* k, double a, double b, double c, double* conic,
                            double* radius, double* lam) {
    double det = a * c - b * b;
    if (!(det > 0.0) || !(a > 0.0)) return DARBS_CPU_NUMERIC_ERROR;
    double mid = 0.5 * (a + c);
    double disc = sqrt(fmax(0.0, mid * mid - det));
    double l1 = mid + disc, l2 = mid - disc;
    conic[0] = c / det;
    conic[1] = -b / det;
    conic[2] = a / det;
    *radius = ceil(sqrt(k->cutoff) * sqrt(l1));
    if (lam) {
        lam[0] = l1;
        lam[1] = l2;
    }
    return DARBS_CPU_OK;
}

int darbs_cpu_conic_and_radius(const darbs_cpu_kernel* k, int n, const double* cov2,
                               double* conic, double* radius, double* lambda12) {
    for (int i = 0; i < n; ++i) {
        int st = conic_radius_one(k, cov2[3 * i], cov2[3 * i + 1], cov2[3 * i + 2], conic + 3 * i,
                                  radius + i, lambda12 ? lambda12 + 2 * i : NULL);
        if (st) return st;
    }
    return DARBS_CPU_OK;
}

/* Eigen::Quaternion::toRotationMatrix of the normalised quaternion
 * (geometry.cpp:13, :115-116).  q = (w, x, y, z). */
static void quat_to_rot(const double* q, double r[9], double qn[4]) {
    double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    double w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
    if (qn) {
        qn[0] = w;
        qn[1] = x;
        qn[2] = y;
        qn[3] = z;
    }
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

static void mat3_mul(const double* a, const double* b, double* o) {
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            double s = 0.0;
            for (int k = 0; k < 3; ++k) s += a[3 * r + k] * b[3 * k + c];
            o[3 * r + c] = s;
        }
}
static void mat3_t(const double* a, double* o) {
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) o[3 * c + r] = a[3 * r + c];
}

/* camera layout: fx fy cx cy width height w[16] (scene_io.hpp:16-19). */
static void cam_rot(const double* cam, double wr[9]) {
    const double* w = cam + 6;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) wr[3 * r + c] = w[4 * r + c];
}
static void cam_point(const double* cam, const double* mu, double t[3]) {
    const double* w = cam + 6;
    for (int r = 0; r < 3; ++r) {
        double s = 0.0;
        for (int c = 0; c < 3; ++c) s += w[4 * r + c] * mu[c];
        t[r] = s + w[4 * r + 3];
    }
}

/* ewa_jacobian geometry.cpp:29-35, then tj = J * W_rot (geometry.cpp:38, :125) */
static void ewa_tj(const double* cam, const double t[3], double j[6], double tj[6]) {
    double fx = cam[0], fy = cam[1];
    double z = t[2];
    j[0] = fx / z;
    j[1] = 0.0;
    j[2] = -fx * t[0] / (z * z);
    j[3] = 0.0;
    j[4] = fy / z;
    j[5] = -fy * t[1] / (z * z);
    double wr[9];
    cam_rot(cam, wr);
    for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 3; ++c) {
            double s = 0.0;
            for (int k = 0; k < 3; ++k) s += j[3 * r + k] * wr[3 * k + c];
            tj[3 * r + c] = s;
        }
}

void darbs_cpu_realize(int n, const double* raw, double* prims) {
    /* realize fit3d.cpp:17-25; sigmoid fit_common.hpp:40 */
    for (int i = 0; i < n; ++i) {
        const double* q = raw + 14 * (size_t)i;
        double* p = prims + 14 * (size_t)i;
        p[0] = q[0];
        p[1] = q[1];
        p[2] = q[2];
        for (int k = 3; k < 6; ++k) p[k] = exp(q[k]);
        for (int k = 6; k < 10; ++k) p[k] = q[k];
        for (int k = 10; k < 14; ++k) p[k] = 1.0 / (1.0 + exp(-q[k]));
    }
}

int darbs_cpu_project(const darbs_cpu_kernel* k, double psi, double dilation, int n,
                      const double* prims, const double* camera, int32_t* valid, double* mu2,
                      double* cov2, double* conic, double* radius, double* depth) {
    for (int i = 0; i < n; ++i) {
        const double* p = prims + 14 * (size_t)i;
        /* project_point geometry.cpp:20-27 */
        double t[3];
        cam_point(camera, p, t);
        if (t[2] <= 0.01) { /* kNearPlane geometry.hpp:55 */
            valid[i] = 0;
            mu2[2 * i] = mu2[2 * i + 1] = 0.0;
            cov2[3 * i] = cov2[3 * i + 1] = cov2[3 * i + 2] = 0.0;
            conic[3 * i] = conic[3 * i + 1] = conic[3 * i + 2] = 0.0;
            radius[i] = 0.0;
            depth[i] = 0.0;
            continue;
        }
        valid[i] = 1;
        mu2[2 * i] = camera[0] * t[0] / t[2] + camera[2];
        mu2[2 * i + 1] = camera[1] * t[1] / t[2] + camera[3];
        depth[i] = t[2];
        /* covariance_from_scale_rot geometry.cpp:9-18 */
        const double* s = p + 3;
        if (!(fmin(s[0], fmin(s[1], s[2])) > 0.0)) return DARBS_CPU_INVALID_PARAMETER;
        double r[9], rd[9], rt[9], m[9], sig[9];
        quat_to_rot(p + 6, r, NULL);
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) rd[3 * a + b] = r[3 * a + b] * (s[b] * s[b]);
        mat3_t(r, rt);
        mat3_mul(rd, rt, m);
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) sig[3 * a + b] = 0.5 * (m[3 * a + b] + m[3 * b + a]);
        /* project_covariance geometry.cpp:37-41 */
        double j[6], tj[6], ts[6];
        ewa_tj(camera, t, j, tj);
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 3; ++b) {
                double acc = 0.0;
                for (int c = 0; c < 3; ++c) acc += tj[3 * a + c] * sig[3 * c + b];
                ts[3 * a + b] = acc;
            }
        double raw[4];
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b) {
                double acc = 0.0;
                for (int c = 0; c < 3; ++c) acc += ts[3 * a + c] * tj[3 * b + c];
                raw[2 * a + b] = acc;
            }
        double rxy = 0.5 * (raw[1] + raw[2]);
        /* apply_psi geometry.cpp:43-48 */
        if (!(psi > 0.0)) return DARBS_CPU_INVALID_PARAMETER;
        double ca = psi * raw[0] + dilation * 1.0;
        double cb = psi * rxy + dilation * 0.0;
        double cc = psi * raw[3] + dilation * 1.0;
        cov2[3 * i] = ca;
        cov2[3 * i + 1] = cb;
        cov2[3 * i + 2] = cc;
        int st = conic_radius_one(k, ca, cb, cc, conic + 3 * i, radius + i, NULL);
        if (st) return st;
    }
    return DARBS_CPU_OK;
}

/* rotation_jacobians geometry.cpp:92-107 (row-major 3x3 each, already x2) */
static void rotation_jacobians(const double q[4], double dr[4][9]) {
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

/* backward_projection geometry.cpp:111-168 for one primitive.
 * gcov = (xx, xy, yx, yy). */
static void backward_projection_one(double psi, const double* gcov, const double* gmu2,
                                    const double* p, const double* cam, double* d_mu,
                                    double* d_scale, double* d_rot) {
    const double* s = p + 3;
    double r[9], qn[4];
    quat_to_rot(p + 6, r, qn);
    double m[9], mt[9], sigma[9];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) m[3 * a + b] = r[3 * a + b] * s[b]; /* :117 */
    mat3_t(m, mt);
    mat3_mul(m, mt, sigma); /* :118 */

    double wrot[9], t[3], j[6], tj[6];
    cam_rot(cam, wrot);
    cam_point(cam, p, t);
    double z = t[2];
    ewa_tj(cam, t, j, tj);
    double fx = cam[0], fy = cam[1];

    /* :127-131 */
    double gsym[4] = {gcov[0], 0.5 * (gcov[1] + gcov[2]), 0.5 * (gcov[1] + gcov[2]), gcov[3]};
    double graw[4];
    for (int i = 0; i < 4; ++i) graw[i] = psi * gsym[i];
    /* d_sigma = tj^T graw tj */
    double gt[6]; /* graw * tj : 2x3 */
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b) gt[3 * a + b] = graw[2 * a] * tj[b] + graw[2 * a + 1] * tj[3 + b];
    double d_sigma[9];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) d_sigma[3 * a + b] = tj[a] * gt[b] + tj[3 + a] * gt[3 + b];
    /* d_tj = 2 graw tj sigma ; d_j = d_tj wrot^T */
    double d_tj[6], d_j[6];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b) {
            double acc = 0.0;
            for (int c = 0; c < 3; ++c) acc += (2.0 * gt[3 * a + c]) * sigma[3 * c + b];
            d_tj[3 * a + b] = acc;
        }
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b) {
            double acc = 0.0;
            for (int c = 0; c < 3; ++c) acc += d_tj[3 * a + c] * wrot[3 * b + c];
            d_j[3 * a + b] = acc;
        }
    /* :134-145 */
    double d_t[3] = {0, 0, 0};
    double z2 = z * z, z3 = z2 * z;
    d_t[0] += d_j[2] * (-fx / z2);
    d_t[1] += d_j[5] * (-fy / z2);
    d_t[2] += d_j[0] * (-fx / z2) + d_j[4] * (-fy / z2) + d_j[2] * (2.0 * fx * t[0] / z3) +
              d_j[5] * (2.0 * fy * t[1] / z3);
    d_t[0] += gmu2[0] * fx / z;
    d_t[1] += gmu2[1] * fy / z;
    d_t[2] += -gmu2[0] * fx * t[0] / z2 - gmu2[1] * fy * t[1] / z2;
    /* :147 d_mu = wrot^T d_t */
    for (int a = 0; a < 3; ++a)
        d_mu[a] = wrot[a] * d_t[0] + wrot[3 + a] * d_t[1] + wrot[6 + a] * d_t[2];
    /* :150-152 */
    double dss[9], d_m[9], d_r[9];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) dss[3 * a + b] = d_sigma[3 * a + b] + d_sigma[3 * b + a];
    mat3_mul(dss, m, d_m);
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) d_r[3 * a + b] = d_m[3 * a + b] * s[b];
    for (int a = 0; a < 3; ++a)
        d_scale[a] = r[a] * d_m[a] + r[3 + a] * d_m[3 + a] + r[6 + a] * d_m[6 + a];
    /* :154-160 */
    double dr[4][9], d_qn[4];
    rotation_jacobians(qn, dr);
    for (int i = 0; i < 4; ++i) {
        double acc = 0.0;
        for (int e = 0; e < 9; ++e) acc += d_r[e] * dr[i][e];
        d_qn[i] = acc;
    }
    /* :163-166 */
    const double* qraw = p + 6;
    double norm = sqrt(qraw[0] * qraw[0] + qraw[1] * qraw[1] + qraw[2] * qraw[2] + qraw[3] * qraw[3]);
    double qu[4], dot = 0.0;
    for (int i = 0; i < 4; ++i) qu[i] = qraw[i] / norm;
    for (int i = 0; i < 4; ++i) dot += qu[i] * d_qn[i];
    for (int i = 0; i < 4; ++i) d_rot[i] = (d_qn[i] - qu[i] * dot) / norm;
}

void darbs_cpu_backward_projection(double psi, int n, const double* grad_cov2,
                                   const double* grad_mu2, const double* prims,
                                   const double* camera, double* d_mu, double* d_scale,
                                   double* d_rot) {
    for (int i = 0; i < n; ++i) {
        backward_projection_one(psi, grad_cov2 + 4 * (size_t)i, grad_mu2 + 2 * (size_t)i,
                                prims + 14 * (size_t)i, camera, d_mu + 3 * (size_t)i,
                                d_scale + 3 * (size_t)i, d_rot + 4 * (size_t)i);
    }
}

void darbs_cpu_param_grads(double psi, int m, const int32_t* owner, const double* splat_grads,
                           const double* conic, const double* opacity, const double* rgb,
                           const double* prims, const double* camera, double* param_grads) {
    for (int k = 0; k < m; ++k) {
        const double* gi = splat_grads + 9 * (size_t)k; /* SplatGrads order */
        int i = owner[k];
        double* g = param_grads + 14 * (size_t)i;
        const double* p = prims + 14 * (size_t)i;
        /* fit3d.cpp:140-144: gc = [[da, db/2],[db/2, dc]], d_cov2 = -C gc C */
        double gc[4] = {gi[4], 0.5 * gi[5], 0.5 * gi[5], gi[6]};
        double cm[4] = {conic[3 * k], conic[3 * k + 1], conic[3 * k + 1], conic[3 * k + 2]};
        double ncm[4] = {-cm[0], -cm[1], -cm[2], -cm[3]};
        double t1[4], d_cov2[4];
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b) t1[2 * a + b] = ncm[2 * a] * gc[b] + ncm[2 * a + 1] * gc[2 + b];
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b) d_cov2[2 * a + b] = t1[2 * a] * cm[b] + t1[2 * a + 1] * cm[2 + b];
        double d_mu[3], d_scale[3], d_rot[4];
        backward_projection_one(psi, d_cov2, gi + 7, p, camera, d_mu, d_scale, d_rot);
        /* fit3d.cpp:148-158 */
        g[0] += d_mu[0];
        g[1] += d_mu[1];
        g[2] += d_mu[2];
        for (int a = 0; a < 3; ++a) g[3 + a] += d_scale[a] * p[3 + a];
        for (int a = 0; a < 4; ++a) g[6 + a] += d_rot[a];
        g[10] += gi[3] * opacity[k] * (1.0 - opacity[k]);
        for (int c = 0; c < 3; ++c) g[11 + c] += gi[c] * rgb[3 * k + c] * (1.0 - rgb[3 * k + c]);
    }
}

/* adam_step optim.hpp:24-39 */
int darbs_cpu_adam_step(int64_t dim, double* params, const double* grads, double* m, double* v,
                        const double* lrs, int t) {
    const double b1 = 0.9, b2 = 0.999, eps = 1e-15; /* optim.hpp:19-21 */
    double bc1 = 1.0 - pow(b1, t);
    double bc2 = 1.0 - pow(b2, t);
    for (int64_t i = 0; i < dim; ++i) {
        m[i] = b1 * m[i] + (1.0 - b1) * grads[i];
        v[i] = b2 * v[i] + (1.0 - b2) * grads[i] * grads[i];
        double mhat = m[i] / bc1;
        double vhat = v[i] / bc2;
        params[i] -= lrs[i] * mhat / (sqrt(vhat) + eps);
    }
    return DARBS_CPU_OK;
}

/* ---------------------------------------------------------- random fixtures */

/* std::mt19937_64 (ISO C++ [rand.predef]) */
typedef struct {
    uint64_t x[312];
    int i;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
    g->x[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->x[i] = 6364136223846793005ULL * (g->x[i - 1] ^ (g->x[i - 1] >> 62)) + (uint64_t)i;
    g->i = 312;
}
static uint64_t mt64_next(mt64* g) {
    if (g->i >= 312) {
        for (int k = 0; k < 312; ++k) {
            uint64_t y = (g->x[k] & 0xFFFFFFFF80000000ULL) | (g->x[(k + 1) % 312] & 0x7FFFFFFFULL);
            g->x[k] = g->x[(k + 156) % 312] ^ (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
        }
        g->i = 0;
    }
    uint64_t y = g->x[g->i++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    return y;
}
/* libstdc++ std::generate_canonical<double,53> over a 64-bit engine followed by
 * uniform_real_distribution's affine map (GCC 13 bits/random.tcc). */
static double mt64_uniform(mt64* g, double a, double b) {
    double c = (double)mt64_next(g) / 18446744073709551616.0;
    if (c >= 1.0) c = nextafter(1.0, 0.0);
    return c * (b - a) + a;
}

static inline double rf(double v, int round_f32) { return round_f32 ? (double)(float)v : v; }

int darbs_cpu_random_scene(const darbs_cpu_kernel* k, int count, int width, int height,
                           uint64_t seed, int round_f32, double* mu2, double* cov2,
                           double* conic, double* radius, double* depth, double* opacity,
                           double* rgb) {
    /* random_scene benchmarks/bench.cpp:20-46 (same distributions as
     * tests/test_rasterizer.cpp:26-46), draw order as bench.cpp:31-41. */
    mt64 g;
    mt64_seed(&g, seed);
    for (int i = 0; i < count; ++i) {
        double a = mt64_uniform(&g, 0.6, 12.0);
        double c = mt64_uniform(&g, 0.6, 12.0);
        double b = mt64_uniform(&g, -0.6, 0.6) * sqrt(a * c);
        double mx = mt64_uniform(&g, -5.0, width + 5.0);
        double my = mt64_uniform(&g, -5.0, height + 5.0);
        a = rf(a, round_f32);
        b = rf(b, round_f32);
        c = rf(c, round_f32);
        cov2[3 * (size_t)i] = a;
        cov2[3 * (size_t)i + 1] = b;
        cov2[3 * (size_t)i + 2] = c;
        mu2[2 * (size_t)i] = rf(mx, round_f32);
        mu2[2 * (size_t)i + 1] = rf(my, round_f32);
        double cn[3], rad;
        int st = conic_radius_one(k, a, b, c, cn, &rad, NULL);
        if (st) return st;
        for (int e = 0; e < 3; ++e) conic[3 * (size_t)i + e] = rf(cn[e], round_f32);
        radius[i] = rad;
        depth[i] = rf(mt64_uniform(&g, 0.5, 9.5), round_f32);
        opacity[i] = rf(mt64_uniform(&g, 0.1, 0.95), round_f32);
        for (int e = 0; e < 3; ++e) rgb[3 * (size_t)i + e] = rf(mt64_uniform(&g, 0.0, 1.0), round_f32);
    }
    return DARBS_CPU_OK;
}

void darbs_cpu_random_image_grad(int width, int height, uint64_t seed, int round_f32,
                                 double* grad_image) {
    mt64 g;
    mt64_seed(&g, seed);
    size_t n = (size_t)width * height * 3;
    for (size_t i = 0; i < n; ++i) grad_image[i] = rf(mt64_uniform(&g, -1.0, 1.0), round_f32);
}

void darbs_cpu_random_image(int width, int height, uint64_t seed, int round_f32, double* rgb) {
    mt64 g;
    mt64_seed(&g, seed);
    size_t n = (size_t)width * height * 3;
    for (size_t i = 0; i < n; ++i) rgb[i] = rf(mt64_uniform(&g, 0.0, 1.0), round_f32);
}

/* ------------------------------------------------------------------- loss */
/* loss.cpp: 11-tap Gaussian window sigma 1.5 (:13-32), mirror padding (:35-41), separable
 * moment filters (:47-74, :105-108), their adjoints (:76-103, :112-115), ssim_terms (:124-140),
 * ssim (:144-171), loss_total (:173-230). */
enum { LOSS_WIN = 11, LOSS_HALF = 5 };

static const double* loss_window(void) { /* loss.cpp:19-32 */
    static double w[LOSS_WIN];
    static int ready = 0;
    if (!ready) {
        double sum = 0.0;
        for (int i = 0; i < LOSS_WIN; ++i) {
            double d = i - LOSS_HALF;
            w[i] = exp(-d * d / (2.0 * 1.5 * 1.5));
            sum += w[i];
        }
        for (int i = 0; i < LOSS_WIN; ++i) w[i] /= sum;
        ready = 1;
    }
    return w;
}

static int loss_reflect(int i, int n) { /* loss.cpp:35-41 */
    while (i < 0 || i >= n) {
        if (i < 0) i = -i - 1;
        if (i >= n) i = 2 * n - 1 - i;
    }
    return i;
}

/* filter_2d loss.cpp:105-108: rows first into tmp, then columns. */
static void loss_filter2d(const double* in, double* out, double* tmp, int w, int h) {
    const double* k = loss_window();
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            double acc = 0.0;
            for (int d = -LOSS_HALF; d <= LOSS_HALF; ++d)
                acc += k[d + LOSS_HALF] * in[(size_t)y * w + loss_reflect(x + d, w)];
            tmp[(size_t)y * w + x] = acc;
        }
    for (int x = 0; x < w; ++x)
        for (int y = 0; y < h; ++y) {
            double acc = 0.0;
            for (int d = -LOSS_HALF; d <= LOSS_HALF; ++d)
                acc += k[d + LOSS_HALF] * tmp[(size_t)loss_reflect(y + d, h) * w + x];
            out[(size_t)y * w + x] = acc;
        }
}

/* scatter_2d loss.cpp:112-115: the transposes in reverse order (columns, then rows). */
static void loss_scatter2d(const double* in, double* out, double* tmp, int w, int h) {
    const double* k = loss_window();
    size_t np = (size_t)w * h;
    for (size_t i = 0; i < np; ++i) tmp[i] = 0.0;
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            double v = in[(size_t)y * w + x];
            if (v == 0.0) continue;
            for (int d = -LOSS_HALF; d <= LOSS_HALF; ++d)
                tmp[(size_t)loss_reflect(y + d, h) * w + x] += k[d + LOSS_HALF] * v;
        }
    for (size_t i = 0; i < np; ++i) out[i] = 0.0;
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            double v = tmp[(size_t)y * w + x];
            if (v == 0.0) continue;
            for (int d = -LOSS_HALF; d <= LOSS_HALF; ++d)
                out[(size_t)y * w + loss_reflect(x + d, w)] += k[d + LOSS_HALF] * v;
        }
}

/* ssim_terms loss.cpp:124-140 */
static double loss_ssim_terms(double mu_x, double mu_y, double sxx, double syy, double sxy,
                              double* d_mu_x, double* d_sxx, double* d_sxy) {
    const double c1 = 0.01 * 0.01, c2 = 0.03 * 0.03;
    double var_x = sxx - mu_x * mu_x;
    double var_y = syy - mu_y * mu_y;
    double cov = sxy - mu_x * mu_y;
    double a1 = 2.0 * mu_x * mu_y + c1;
    double a2 = 2.0 * cov + c2;
    double b1 = mu_x * mu_x + mu_y * mu_y + c1;
    double b2 = var_x + var_y + c2;
    double denom = b1 * b2;
    if (d_mu_x)
        *d_mu_x = 2.0 * mu_y * (a2 - a1) / denom - 2.0 * mu_x * a1 * a2 * (b2 - b1) / (denom * denom);
    if (d_sxx) *d_sxx = -a1 * a2 / (b1 * b2 * b2);
    if (d_sxy) *d_sxy = 2.0 * a1 / denom;
    return a1 * a2 / denom;
}

typedef struct {
    double *x, *y, *buf, *tmp, *mu_x, *mu_y, *sxx, *syy, *sxy, *fa, *fb, *fd, *sa, *sb, *sd;
    double* block;
} loss_planes;

static int loss_planes_alloc(loss_planes* p, size_t np) {
    p->block = (double*)malloc(sizeof(double) * 15 * (np ? np : 1));
    if (!p->block) return 0;
    double** f = &p->x;
    for (int i = 0; i < 15; ++i) f[i] = p->block + (size_t)i * np;
    return 1;
}

/* moments of one channel, loss.cpp:150-163 / :206-216 */
static void loss_moments(loss_planes* p, const double* a, const double* b, int c, int w, int h) {
    size_t np = (size_t)w * h;
    for (size_t i = 0; i < np; ++i) {
        p->x[i] = a[i * 3 + c];
        p->y[i] = b[i * 3 + c];
    }
    loss_filter2d(p->x, p->mu_x, p->tmp, w, h);
    loss_filter2d(p->y, p->mu_y, p->tmp, w, h);
    for (size_t i = 0; i < np; ++i) p->buf[i] = p->x[i] * p->x[i];
    loss_filter2d(p->buf, p->sxx, p->tmp, w, h);
    for (size_t i = 0; i < np; ++i) p->buf[i] = p->y[i] * p->y[i];
    loss_filter2d(p->buf, p->syy, p->tmp, w, h);
    for (size_t i = 0; i < np; ++i) p->buf[i] = p->x[i] * p->y[i];
    loss_filter2d(p->buf, p->sxy, p->tmp, w, h);
}

int darbs_cpu_ssim(int width, int height, const double* a, const double* b, double* out) {
    if (width < 0 || height < 0) return DARBS_CPU_INVALID_PARAMETER;
    size_t np = (size_t)width * height;
    loss_planes p;
    if (!loss_planes_alloc(&p, np)) return DARBS_CPU_NUMERIC_ERROR;
    double acc = 0.0;
    for (int c = 0; c < 3; ++c) {
        loss_moments(&p, a, b, c, width, height);
        for (size_t i = 0; i < np; ++i)
            acc += loss_ssim_terms(p.mu_x[i], p.mu_y[i], p.sxx[i], p.syy[i], p.sxy[i], NULL, NULL, NULL);
    }
    free(p.block);
    *out = acc / (3.0 * (double)np);
    return DARBS_CPU_OK;
}

int darbs_cpu_loss_total(int width, int height, const double* rendered, const double* target,
                         double lambda, double out[3], double* grad) {
    if (width < 0 || height < 0) return DARBS_CPU_INVALID_PARAMETER;
    size_t np = (size_t)width * height, n = 3 * np;
    loss_planes p;
    if (!loss_planes_alloc(&p, np)) return DARBS_CPU_NUMERIC_ERROR;
    double l1 = 0.0;
    for (size_t i = 0; i < n; ++i) { /* loss.cpp:183-188 */
        double d = rendered[i] - target[i];
        l1 += fabs(d);
        if (grad) grad[i] = (1.0 - lambda) * (double)((d > 0) - (d < 0)) / (double)n;
    }
    l1 /= (double)n;
    double ssim_acc = 0.0;
    const double scale = -0.5 * lambda / (double)n; /* loss.cpp:196 */
    for (int c = 0; c < 3; ++c) {
        loss_moments(&p, rendered, target, c, width, height);
        for (size_t i = 0; i < np; ++i) { /* loss.cpp:210-216 */
            double da, db, dd;
            ssim_acc += loss_ssim_terms(p.mu_x[i], p.mu_y[i], p.sxx[i], p.syy[i], p.sxy[i], &da, &db, &dd);
            p.fa[i] = scale * da;
            p.fb[i] = scale * db;
            p.fd[i] = scale * dd;
        }
        if (lambda == 0.0 || !grad) continue;
        loss_scatter2d(p.fa, p.sa, p.tmp, width, height);
        loss_scatter2d(p.fb, p.sb, p.tmp, width, height);
        loss_scatter2d(p.fd, p.sd, p.tmp, width, height);
        for (size_t i = 0; i < np; ++i) /* loss.cpp:222-224 */
            grad[i * 3 + c] += p.sa[i] + 2.0 * p.x[i] * p.sb[i] + p.y[i] * p.sd[i];
    }
    free(p.block);
    double mean_ssim = ssim_acc / (double)n;
    out[1] = l1;
    out[2] = 0.5 * (1.0 - mean_ssim);
    out[0] = (1.0 - lambda) * out[1] + lambda * out[2];
    return DARBS_CPU_OK;
}

/* ------------------------------------------------------------- parallel_for */

/* parallel_for parallel.hpp:19-33: `threads` workers, static round-robin
 * striding i = t, t+threads, ...; threads <= 0 -> hardware concurrency. */
typedef void (*work_fn)(size_t item, void* ctx);
typedef struct {
    work_fn fn;
    void* ctx;
    size_t count;
    int t, threads;
} worker_arg;

static void* worker_main(void* p) {
    worker_arg* a = (worker_arg*)p;
    for (size_t i = (size_t)a->t; i < a->count; i += (size_t)a->threads) a->fn(i, a->ctx);
    return NULL;
}

static int resolve_threads(int requested) {
    if (requested > 0) return requested;
    long hw = sysconf(_SC_NPROCESSORS_ONLN);
    return hw <= 0 ? 1 : (int)hw;
}

static void parallel_for(size_t count, int threads, work_fn fn, void* ctx) {
    threads = resolve_threads(threads);
    if ((size_t)threads > count) threads = (int)count;
    if (threads <= 1) {
        for (size_t i = 0; i < count; ++i) fn(i, ctx);
        return;
    }
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    worker_arg* args = (worker_arg*)malloc(sizeof(worker_arg) * (size_t)threads);
    for (int t = 0; t < threads; ++t) {
        args[t].fn = fn;
        args[t].ctx = ctx;
        args[t].count = count;
        args[t].t = t;
        args[t].threads = threads;
        pthread_create(&th[t], NULL, worker_main, &args[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
    free(args);
}

/* --------------------------------------------------------------- rasterizer */

#define TILE 16                  /* kTileSize rasterizer.hpp:11 */
#define ALPHA_CLAMP 0.99         /* kAlphaClamp :12 */
#define ALPHA_SKIP (1.0 / 255.0) /* kAlphaSkip :13 */
#define T_FLOOR 1e-4             /* kTransmittanceFloor :14 */

static inline int conic_finite(const double* c) { /* rasterizer.cpp:15-17 */
    return isfinite(c[0]) && isfinite(c[1]) && isfinite(c[2]);
}
static inline double conic_dm2(const double* c, double dx, double dy) { /* rasterizer.cpp:19-21 */
    return c[0] * dx * dx + 2.0 * c[1] * dx * dy + c[2] * dy * dy;
}

typedef struct {
    const double* depth;
} depth_cmp_ctx;
typedef struct {
    double depth;
    int32_t idx;
} depth_item;

static int depth_item_cmp(const void* a, const void* b) {
    const depth_item* x = (const depth_item*)a;
    const depth_item* y = (const depth_item*)b;
    /* std::stable_sort by depth (rasterizer.cpp:33) == total order (depth, idx) */
    if (x->depth < y->depth) return -1;
    if (y->depth < x->depth) return 1;
    return (x->idx > y->idx) - (x->idx < y->idx);
}

static void tile_rect(const double* mu2, double radius, int tiles_x, int tiles_y, int* x0, int* y0,
                      int* x1, int* y1) {
    /* rasterizer.cpp:40-45 */
    int a = (int)floor((mu2[0] - radius) / TILE);
    int b = (int)floor((mu2[1] - radius) / TILE);
    int c = (int)floor((mu2[0] + radius) / TILE);
    int d = (int)floor((mu2[1] + radius) / TILE);
    *x0 = a > 0 ? a : 0;
    *y0 = b > 0 ? b : 0;
    *x1 = c < tiles_x - 1 ? c : tiles_x - 1;
    *y1 = d < tiles_y - 1 ? d : tiles_y - 1;
}

typedef struct {
    int tiles_x, tiles_y;
    int64_t* offsets; /* tiles+1 */
    int32_t* list;    /* K */
} bins_t;

/* bin_splats rasterizer.cpp:25-53 as CSR: a counting pass then a fill pass in
 * depth order, which yields exactly the push_back order of :46-50. */
static int bins_build(bins_t* bins, int n, const double* mu2, const double* conic,
                      const double* radius, const double* depth, int width, int height,
                      int32_t* depth_order_out) {
    bins->tiles_x = (width + TILE - 1) / TILE;
    bins->tiles_y = (height + TILE - 1) / TILE;
    size_t tiles = (size_t)bins->tiles_x * bins->tiles_y;
    bins->offsets = (int64_t*)calloc(tiles + 1, sizeof(int64_t));
    bins->list = NULL;
    depth_item* order = (depth_item*)malloc(sizeof(depth_item) * (size_t)(n > 0 ? n : 1));
    for (int i = 0; i < n; ++i) {
        order[i].depth = depth[i];
        order[i].idx = i;
    }
    qsort(order, (size_t)n, sizeof(depth_item), depth_item_cmp);
    if (depth_order_out)
        for (int i = 0; i < n; ++i) depth_order_out[i] = order[i].idx;

    for (int pass = 0; pass < 2; ++pass) {
        int64_t* cursor = NULL;
        if (pass == 1) {
            /* exclusive scan of counts held in offsets[t+1] */
            for (size_t t = 0; t < tiles; ++t) bins->offsets[t + 1] += bins->offsets[t];
            bins->list = (int32_t*)malloc(sizeof(int32_t) * (size_t)(bins->offsets[tiles] + 1));
            cursor = (int64_t*)malloc(sizeof(int64_t) * (tiles + 1));
            memcpy(cursor, bins->offsets, sizeof(int64_t) * (tiles + 1));
        }
        for (int r = 0; r < n; ++r) {
            int idx = order[r].idx;
            if (!conic_finite(conic + 3 * (size_t)idx) || !isfinite(radius[idx])) continue; /* :39 */
            int x0, y0, x1, y1;
            tile_rect(mu2 + 2 * (size_t)idx, radius[idx], bins->tiles_x, bins->tiles_y, &x0, &y0, &x1,
                      &y1);
            for (int ty = y0; ty <= y1; ++ty)
                for (int tx = x0; tx <= x1; ++tx) {
                    size_t t = (size_t)ty * bins->tiles_x + tx;
                    if (pass == 0)
                        bins->offsets[t + 1]++;
                    else
                        bins->list[cursor[t]++] = idx;
                }
        }
        free(cursor);
    }
    free(order);
    return 0;
}

int64_t darbs_cpu_bin(int n, const double* mu2, const double* conic, const double* radius,
                      const double* depth, int width, int height, int64_t* tile_offsets,
                      int32_t* point_list, int64_t capacity, int32_t* depth_order) {
    bins_t b;
    bins_build(&b, n, mu2, conic, radius, depth, width, height, depth_order);
    size_t tiles = (size_t)b.tiles_x * b.tiles_y;
    int64_t k = b.offsets[tiles];
    if (tile_offsets) memcpy(tile_offsets, b.offsets, sizeof(int64_t) * (tiles + 1));
    if (point_list && k <= capacity) memcpy(point_list, b.list, sizeof(int32_t) * (size_t)k);
    free(b.offsets);
    free(b.list);
    return k;
}

/* BlendAux rasterizer.hpp:27-37 */
typedef struct {
    int width, height, n;
    double background[3];
    bins_t bins;
    double* t_final;
    int32_t* processed;
    int32_t* contributors;
    int skipped;
} aux_t;

typedef struct {
    const darbs_cpu_kernel* k;
    const double *mu2, *conic, *opacity, *rgb;
    aux_t* aux;
    double* image;
    /* backward only */
    const double* grad_image;
    double** tile_grads;
} raster_ctx;

/* forward tile body rasterizer.cpp:77-110 */
static void forward_tile(size_t t, void* vctx) {
    raster_ctx* c = (raster_ctx*)vctx;
    aux_t* aux = c->aux;
    int width = aux->width, height = aux->height;
    int tx = (int)t % aux->bins.tiles_x;
    int ty = (int)t / aux->bins.tiles_x;
    const int32_t* list = aux->bins.list + aux->bins.offsets[t];
    int64_t len = aux->bins.offsets[t + 1] - aux->bins.offsets[t];
    int px0 = tx * TILE, py0 = ty * TILE;
    int px1 = width < px0 + TILE ? width : px0 + TILE;
    int py1 = height < py0 + TILE ? height : py0 + TILE;
    for (int y = py0; y < py1; ++y) {
        for (int x = px0; x < px1; ++x) {
            double cx = x + 0.5, cy = y + 0.5;
            double T = 1.0;
            double col[3] = {0, 0, 0};
            int done = 0, contrib = 0;
            for (int64_t li = 0; li < len; ++li) {
                int idx = list[li];
                ++done;
                double dm2 = conic_dm2(c->conic + 3 * (size_t)idx, cx - c->mu2[2 * (size_t)idx],
                                       cy - c->mu2[2 * (size_t)idx + 1]);
                if (dm2 < 0.0) continue;
                double w, dw;
                kernel_eval(c->k, dm2, &w, &dw);
                double alpha = fmin(ALPHA_CLAMP, c->opacity[idx] * w);
                if (alpha < ALPHA_SKIP) continue;
                for (int ch = 0; ch < 3; ++ch) col[ch] += c->rgb[3 * (size_t)idx + ch] * (alpha * T);
                T *= 1.0 - alpha;
                ++contrib;
                if (T < T_FLOOR) break;
            }
            size_t p = (size_t)y * width + x;
            for (int ch = 0; ch < 3; ++ch) col[ch] += aux->background[ch] * T;
            aux->t_final[p] = T;
            aux->processed[p] = done;
            aux->contributors[p] = contrib;
            for (int ch = 0; ch < 3; ++ch) c->image[p * 3 + ch] = col[ch];
        }
    }
}

void* darbs_cpu_forward(const darbs_cpu_kernel* k, int n, const double* mu2, const double* conic,
                        const double* radius, const double* depth, const double* opacity,
                        const double* rgb, int width, int height, const double* background,
                        int threads, double* image, double* t_final, int32_t* processed,
                        int32_t* contributors, int32_t* skipped_nonfinite) {
    /* forward rasterizer.cpp:55-112 */
    aux_t* aux = (aux_t*)calloc(1, sizeof(aux_t));
    size_t px = (size_t)width * height;
    aux->width = width;
    aux->height = height;
    aux->n = n;
    memcpy(aux->background, background, sizeof(double) * 3);
    bins_build(&aux->bins, n, mu2, conic, radius, depth, width, height, NULL);
    aux->t_final = (double*)malloc(sizeof(double) * (px ? px : 1));
    aux->processed = (int32_t*)calloc(px ? px : 1, sizeof(int32_t));
    aux->contributors = (int32_t*)calloc(px ? px : 1, sizeof(int32_t));
    for (size_t p = 0; p < px; ++p) aux->t_final[p] = 1.0;
    int skipped = 0;
    for (int i = 0; i < n; ++i)
        if (!conic_finite(conic + 3 * (size_t)i) || !isfinite(radius[i])) skipped++; /* :69-73 */
    aux->skipped = skipped;

    double* img = image ? image : (double*)malloc(sizeof(double) * (px ? px : 1) * 3);
    raster_ctx ctx = {k, mu2, conic, opacity, rgb, aux, img, NULL, NULL};
    parallel_for((size_t)aux->bins.tiles_x * aux->bins.tiles_y, threads, forward_tile, &ctx);
    if (!image) free(img);
    if (t_final) memcpy(t_final, aux->t_final, sizeof(double) * px);
    if (processed) memcpy(processed, aux->processed, sizeof(int32_t) * px);
    if (contributors) memcpy(contributors, aux->contributors, sizeof(int32_t) * px);
    if (skipped_nonfinite) *skipped_nonfinite = skipped;
    return aux;
}

void darbs_cpu_forward_free(void* handle) {
    aux_t* aux = (aux_t*)handle;
    if (!aux) return;
    free(aux->bins.offsets);
    free(aux->bins.list);
    free(aux->t_final);
    free(aux->processed);
    free(aux->contributors);
    free(aux);
}

int darbs_cpu_oracle_forward(const darbs_cpu_kernel* k, int n, const double* mu2,
                             const double* conic, const double* radius, const double* depth,
                             const double* opacity, const double* rgb, int width, int height,
                             const double* background, double* image) {
    /* oracle_forward rasterizer.cpp:114-145 */
    depth_item* order = (depth_item*)malloc(sizeof(depth_item) * (size_t)(n > 0 ? n : 1));
    for (int i = 0; i < n; ++i) {
        order[i].depth = depth[i];
        order[i].idx = i;
    }
    qsort(order, (size_t)n, sizeof(depth_item), depth_item_cmp);
    for (int y = 0; y < height; ++y) {
        for (int x = 0; x < width; ++x) {
            double cx = x + 0.5, cy = y + 0.5, T = 1.0;
            double col[3] = {0, 0, 0};
            for (int r = 0; r < n; ++r) {
                int idx = order[r].idx;
                if (!conic_finite(conic + 3 * (size_t)idx) || !isfinite(radius[idx])) continue;
                double dm2 = conic_dm2(conic + 3 * (size_t)idx, cx - mu2[2 * (size_t)idx],
                                       cy - mu2[2 * (size_t)idx + 1]);
                if (dm2 < 0.0) continue;
                double w, dw;
                kernel_eval(k, dm2, &w, &dw);
                double alpha = fmin(ALPHA_CLAMP, opacity[idx] * w);
                if (alpha < ALPHA_SKIP) continue;
                for (int ch = 0; ch < 3; ++ch) col[ch] += rgb[3 * (size_t)idx + ch] * (alpha * T);
                T *= 1.0 - alpha;
                if (T < T_FLOOR) break;
            }
            size_t p = (size_t)y * width + x;
            for (int ch = 0; ch < 3; ++ch) image[p * 3 + ch] = col[ch] + background[ch] * T;
        }
    }
    free(order);
    return DARBS_CPU_OK;
}

/* backward tile body rasterizer.cpp:161-216; per-tile buffer of 9 doubles per
 * list position (SplatGrads order). */
static void backward_tile(size_t t, void* vctx) {
    raster_ctx* c = (raster_ctx*)vctx;
    aux_t* aux = c->aux;
    const int32_t* list = aux->bins.list + aux->bins.offsets[t];
    int64_t len = aux->bins.offsets[t + 1] - aux->bins.offsets[t];
    if (len == 0) return;
    double* local = (double*)calloc((size_t)len * 9, sizeof(double));
    c->tile_grads[t] = local;
    int tx = (int)t % aux->bins.tiles_x;
    int ty = (int)t / aux->bins.tiles_x;
    int px0 = tx * TILE, py0 = ty * TILE;
    int px1 = aux->width < px0 + TILE ? aux->width : px0 + TILE;
    int py1 = aux->height < py0 + TILE ? aux->height : py0 + TILE;
    for (int y = py0; y < py1; ++y) {
        for (int x = px0; x < px1; ++x) {
            size_t p = (size_t)y * aux->width + x;
            int done = aux->processed[p];
            if (done == 0) continue;
            double cx = x + 0.5, cy = y + 0.5;
            const double* g = c->grad_image + p * 3;
            double T = aux->t_final[p];
            double behind[3] = {aux->background[0] * T, aux->background[1] * T,
                                aux->background[2] * T};
            for (int li = done - 1; li >= 0; --li) {
                int idx = list[li];
                const double* cn = c->conic + 3 * (size_t)idx;
                const double* col = c->rgb + 3 * (size_t)idx;
                double dx = cx - c->mu2[2 * (size_t)idx], dy = cy - c->mu2[2 * (size_t)idx + 1];
                double dm2 = conic_dm2(cn, dx, dy);
                if (dm2 < 0.0) continue;
                double w, dw;
                kernel_eval(c->k, dm2, &w, &dw);
                double alpha_raw = c->opacity[idx] * w;
                double alpha = fmin(ALPHA_CLAMP, alpha_raw);
                if (alpha < ALPHA_SKIP) continue;
                double t_before = T / (1.0 - alpha);
                double* sg = local + 9 * (size_t)li;
                for (int ch = 0; ch < 3; ++ch) sg[ch] += g[ch] * (alpha * t_before);
                double d_alpha = 0.0;
                for (int ch = 0; ch < 3; ++ch)
                    d_alpha += g[ch] * (col[ch] * t_before - behind[ch] / (1.0 - alpha));
                if (alpha_raw < ALPHA_CLAMP) {
                    sg[3] += d_alpha * w;
                    double d_dm2 = d_alpha * c->opacity[idx] * dw;
                    sg[4] += d_dm2 * dx * dx;
                    sg[5] += d_dm2 * 2.0 * dx * dy;
                    sg[6] += d_dm2 * dy * dy;
                    sg[7] += -d_dm2 * (2.0 * cn[0] * dx + 2.0 * cn[1] * dy);
                    sg[8] += -d_dm2 * (2.0 * cn[1] * dx + 2.0 * cn[2] * dy);
                }
                for (int ch = 0; ch < 3; ++ch) behind[ch] += col[ch] * (alpha * t_before);
                T = t_before;
            }
        }
    }
}

int darbs_cpu_backward(void* handle, const darbs_cpu_kernel* k, int grad_width, int grad_height,
                       const double* grad_image, int n, const double* mu2, const double* conic,
                       const double* opacity, const double* rgb, int threads, double* grads) {
    aux_t* aux = (aux_t*)handle;
    if (!aux || grad_width != aux->width || grad_height != aux->height || n != aux->n)
        return DARBS_CPU_CONTRACT_VIOLATION; /* rasterizer.cpp:151-154 */
    size_t tiles = (size_t)aux->bins.tiles_x * aux->bins.tiles_y;
    double** tile_grads = (double**)calloc(tiles ? tiles : 1, sizeof(double*));
    raster_ctx ctx = {k, mu2, conic, opacity, rgb, aux, NULL, grad_image, tile_grads};
    parallel_for(tiles, threads, backward_tile, &ctx);
    /* fixed-order reduction rasterizer.cpp:218-232 */
    memset(grads, 0, sizeof(double) * 9 * (size_t)n);
    for (size_t t = 0; t < tiles; ++t) {
        if (!tile_grads[t]) continue;
        const int32_t* list = aux->bins.list + aux->bins.offsets[t];
        int64_t len = aux->bins.offsets[t + 1] - aux->bins.offsets[t];
        for (int64_t li = 0; li < len; ++li) {
            double* dst = grads + 9 * (size_t)list[li];
            const double* src = tile_grads[t] + 9 * (size_t)li;
            for (int e = 0; e < 9; ++e) dst[e] += src[e];
        }
        free(tile_grads[t]);
    }
    free(tile_grads);
    return DARBS_CPU_OK;
}
