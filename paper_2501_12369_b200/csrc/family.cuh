// family.cuh — device functors of the DARBF reconstruction-kernel family.
//
// Restates darbs::eval (reference src/kernel.cpp:127-164, family_fu :73-104,
// center_dweight :109-123) in two forms:
//   * fam_eval<FAM>(m)   FP32 closed forms on the scaled squared distance
//                         m = scale * dm2, one or two MUFU ops each;
//   * eval_exact(kp,dm2) FP64, branch for branch as the reference writes it; used
//                         for decisions inside the FP32 guard band and by the
//                         parity tests of darbs_cuda_eval.
#pragma once

#include "common.cuh"

namespace darbs_b200 {

static constexpr float kAlphaClampF = 0.99f;
static constexpr float kAlphaSkipF = 1.0f / 255.0f;
static constexpr float kTFloorF = 1e-4f;
static constexpr double kAlphaClampD = 0.99;
static constexpr double kAlphaSkipD = 1.0 / 255.0;
static constexpr double kPiD = 3.14159265358979323846;

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rsqrt_approx(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float sqrt_approx(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// scale such that m = scale * dm2 feeds the closed form directly.
__host__ __device__ inline double family_scale(int fam, double xi) {
    switch (fam) {
        case FAM_GAUSS2:
            return 1.4426950408889634 / xi;  // log2(e)/xi : w = 2^-m
        case FAM_HCOS2:
            return 1.0 / xi;                 // w = cos(m)
        case FAM_RCOS1:
            return 1.0 / (xi * xi);          // w = .5 + .5 cos(sqrt(m))
        case FAM_IMQ:
            return 1.0 / xi;                 // w = rsqrt(m + 1)
        case FAM_MSINC1:
            return 1.0 / (xi * xi);          // w = sin(sqrt(m)) / sqrt(m)
        default:
            return 1.0;
    }
}

// sin(sqrt(m))/sqrt(m) = sum_k (-m)^k / (2k+1)! on the main lobe m in [0, pi^2]: an entire
// function of m, so the single-lobe modulus sinc (|sin u| = sin u on [0, pi], kernel.cpp:87-98)
// needs neither the square root nor a trigonometric call.  Eleven terms leave 2e-10 at m = pi^2;
// the terms never exceed 1.7, so Horner in FP32 is good to ~2e-7 absolute.
__device__ __forceinline__ float msinc_poly(float m) {
    float p = 1.9572941063391263e-20f;                            //  1/21!
    p = fmaf(p, m, -8.2206352466243297e-18f);                     // -1/19!
    p = fmaf(p, m, 2.8114572543455208e-15f);                      //  1/17!
    p = fmaf(p, m, -7.6471637318198165e-13f);                     // -1/15!
    p = fmaf(p, m, 1.6059043836821613e-10f);                      //  1/13!
    p = fmaf(p, m, -2.5052108385441719e-08f);                     // -1/11!
    p = fmaf(p, m, 2.7557319223985893e-06f);                      //  1/9!
    p = fmaf(p, m, -1.9841269841269841e-04f);                     // -1/7!
    p = fmaf(p, m, 8.3333333333333333e-03f);                      //  1/5!
    p = fmaf(p, m, -1.6666666666666666e-01f);                     // -1/3!
    return fmaf(p, m, 1.0f);
}
// d/dm of the series: sum_k (-1)^k k m^(k-1) / (2k+1)!
__device__ __forceinline__ float msinc_dpoly(float m) {
    float p = 10.0f * 1.9572941063391263e-20f;
    p = fmaf(p, m, -9.0f * 8.2206352466243297e-18f);
    p = fmaf(p, m, 8.0f * 2.8114572543455208e-15f);
    p = fmaf(p, m, -7.0f * 7.6471637318198165e-13f);
    p = fmaf(p, m, 6.0f * 1.6059043836821613e-10f);
    p = fmaf(p, m, -5.0f * 2.5052108385441719e-08f);
    p = fmaf(p, m, 4.0f * 2.7557319223985893e-06f);
    p = fmaf(p, m, -3.0f * 1.9841269841269841e-04f);
    p = fmaf(p, m, 2.0f * 8.3333333333333333e-03f);
    return fmaf(p, m, -1.6666666666666666e-01f);
}

// FP32 weight and derivative with respect to m (NOT dm2) for m inside the
// support.  Callers zero the result past the cutoff.
template <int FAM>
__device__ __forceinline__ void fam_eval(float m, float& w, float& dwdm) {
    if constexpr (FAM == FAM_GAUSS2) {
        w = ex2_approx(-m);
        dwdm = -0.6931471805599453f * w;
    } else if constexpr (FAM == FAM_HCOS2) {
        w = __cosf(m);
        dwdm = -__sinf(m);
    } else if constexpr (FAM == FAM_RCOS1) {
        float u = sqrt_approx(fmaxf(m, 0.f));  // FP32 rounding can leave m a hair below zero
        w = fmaf(0.5f, __cosf(u), 0.5f);
        // d/dm [.5 + .5 cos(sqrt m)] = -.25 sin(u)/u  -> -.25 as u -> 0 (kernel.cpp:115-116)
        dwdm = (m < 1e-12f) ? -0.25f : -0.25f * __sinf(u) * rsqrt_approx(m);
    } else if constexpr (FAM == FAM_IMQ) {
        float r = rsqrt_approx(m + 1.0f);
        w = r;
        dwdm = -0.5f * r * r * r;
    } else if constexpr (FAM == FAM_MSINC1) {
        w = fminf(fmaxf(msinc_poly(m), 0.f), 1.f);  // kernel.cpp:161 clamps f to [0, 1]
        dwdm = msinc_dpoly(m);
    } else {
        w = 0.f;
        dwdm = 0.f;
    }
}

template <int FAM>
__device__ __forceinline__ float fam_weight(float m) {
    if constexpr (FAM == FAM_GAUSS2) {
        return ex2_approx(-m);
    } else if constexpr (FAM == FAM_HCOS2) {
        return __cosf(m);
    } else if constexpr (FAM == FAM_RCOS1) {
        return fmaf(0.5f, __cosf(sqrt_approx(fmaxf(m, 0.f))), 0.5f);
    } else if constexpr (FAM == FAM_IMQ) {
        return rsqrt_approx(m + 1.0f);
    } else if constexpr (FAM == FAM_MSINC1) {
        return fminf(fmaxf(msinc_poly(m), 0.f), 1.f);
    } else {
        return 0.f;
    }
}

// u_limit kernel.cpp:27-38 / family_fu kernel.cpp:73-104 in FP64.
__device__ inline void family_fu_exact(int family, double u, double& f, double& df) {
    switch (family) {
        case DARBS_GAUSSIAN:
            f = exp(-u);
            df = -f;
            return;
        case DARBS_HALF_COSINE:
            f = cos(u);
            df = -sin(u);
            return;
        case DARBS_RAISED_COSINE:
            f = 0.5 + 0.5 * cos(u);
            df = -0.5 * sin(u);
            return;
        case DARBS_MODULUS_SINC: {
            if (u < 1e-8) {
                f = 1.0 - u * u / 6.0;
                df = -u / 3.0;
                return;
            }
            double s = sin(u);
            double sgn = (double)((s > 0.0) - (s < 0.0));
            f = fabs(s) / u;
            df = sgn * (u * cos(u) - s) / (u * u);
            return;
        }
        default:
            f = 0.0;
            df = 0.0;
            return;
    }
}

// center_dweight kernel.cpp:109-123
__device__ inline double center_dweight_exact(const KParams& s) {
    switch (s.family) {
        case DARBS_GAUSSIAN:
            return s.beta_d == 2.0 ? -1.0 / s.xi_d : 0.0;
        case DARBS_HALF_COSINE:
            return s.beta_d == 1.0 ? -1.0 / (2.0 * s.xi_d * s.xi_d) : 0.0;
        case DARBS_RAISED_COSINE:
            return s.beta_d == 1.0 ? -1.0 / (4.0 * s.xi_d * s.xi_d) : 0.0;
        case DARBS_MODULUS_SINC:
            return s.beta_d == 1.0 ? -1.0 / (6.0 * s.xi_d * s.xi_d) : 0.0;
        case DARBS_INVERSE_MULTIQUADRATIC:
            return -1.0 / (2.0 * s.xi_d);
    }
    return 0.0;
}

// eval kernel.cpp:127-164 (dm2 >= 0 and finite is the caller's business).
__device__ inline void eval_exact(const KParams& spec, double dm2, double& weight, double& dweight) {
    weight = 0.0;
    dweight = 0.0;
    if (spec.unbounded ? dm2 > spec.cutoff_d : dm2 >= spec.cutoff_d) return;
    if (spec.family == DARBS_INVERSE_MULTIQUADRATIC) {
        double base = dm2 / spec.xi_d + 1.0;
        double r = 1.0 / sqrt(base);
        weight = r;
        dweight = -0.5 * r / (base * spec.xi_d);
        return;
    }
    if (dm2 < 1e-30) {
        double f, df;
        family_fu_exact(spec.family, 0.0, f, df);
        weight = f;
        dweight = center_dweight_exact(spec);
        return;
    }
    double u = (spec.beta_d == 2.0) ? dm2 / spec.xi_d : pow(dm2, 0.5 * spec.beta_d) / spec.xi_d;
    double f, df;
    family_fu_exact(spec.family, u, f, df);
    double du = (spec.beta_d == 2.0)
                    ? 1.0 / spec.xi_d
                    : 0.5 * spec.beta_d * pow(dm2, 0.5 * spec.beta_d - 1.0) / spec.xi_d;
    weight = fmin(fmax(f, 0.0), 1.0);
    dweight = df * du;
}

// Largest dm2 at which a splat of opacity o can still reach alpha >= 1/255
// (rasterizer.cpp:94), intersected with the render cutoff — the per-splat
// decision boundary in dm2 units.  The monotone single-lobe families invert in
// closed form; FAM_GENERIC keeps the cutoff (used for culling only).  Returns
// a negative value when the splat can never contribute and NaN when the
// decision must always be taken by the FP64 path.
__device__ inline double family_threshold(const KParams& kp, double o) {
    if (!(o == o)) return nan("");
    if (!(o > 0.0)) return -1.0;
    double t = 1.0 / (255.0 * o);  // weight needed for alpha == 1/255
    double thr;
    switch (kp.fam) {
        case FAM_GAUSS2:
            thr = -kp.xi_d * log(t);
            break;
        case FAM_HCOS2:
            thr = t > 1.0 ? -1.0 : kp.xi_d * acos(t);
            break;
        case FAM_RCOS1: {
            double v = 2.0 * t - 1.0;
            if (v > 1.0) {
                thr = -1.0;
            } else if (v <= -1.0) {
                thr = kp.cutoff_d;
            } else {
                double u = kp.xi_d * acos(v);
                thr = u * u;
            }
            break;
        }
        case FAM_IMQ:
            thr = t > 1.0 ? -1.0 : kp.xi_d * (1.0 / (t * t) - 1.0);
            break;
        case FAM_MSINC1: {
            // sin(u)/u = t on [0, pi] (monotone): Newton from the two-term series u0 = sqrt(6 (1 - t)).
            // The result only has to land inside the guard band, where decisions are re-taken exactly.
            if (t > 1.0) {
                thr = -1.0;
            } else {
                double u = fmin(sqrt(6.0 * (1.0 - t)), kPiD);
                for (int it = 0; it < 6 && u > 1e-6; ++it) {
                    const double su = sin(u), cu = cos(u);
                    const double f = su / u - t, df = (u * cu - su) / (u * u);
                    u = fmin(fmax(u - f / df, 0.0), kPiD);
                }
                thr = (kp.xi_d * u) * (kp.xi_d * u);
            }
            break;
        }
        default:
            thr = kp.cutoff_d;
            break;
    }
    return fmin(thr, kp.cutoff_d);
}

}  // namespace darbs_b200
