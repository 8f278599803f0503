/*
 * darbs_cpu.h — C interface of the CPU ORACLE for the DARBF rasterizer hot path.
 *
 * TEST INFRASTRUCTURE, NOT PRODUCT.  Two shared libraries implement this one
 * interface with identical symbol names:
 *
 *   oracle/libdarbs_oracle.so   plain-C FP64 restatement (oracle/darbs_oracle.c),
 *                               every function citing the reference file:line
 *                               it follows; travels to the GPU box.
 *   oracle/_ref/libdarbs_ref.so the reference's OWN sources
 *                               (/root/reference/proj/core/src/{kernel,geometry,
 *                               rasterizer,loss}.cpp, unmodified) compiled against
 *                               oracle/eigen_shim and wrapped by
 *                               oracle/ref_glue.cpp.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load either library, and only as the checker or the timed
 * CPU baseline.  The product (paper_2501_12369_b200/) never links or loads
 * anything under oracle/.
 *
 * All arrays are FP64 (the reference's element type) in structure-of-arrays
 * form.  Status codes match include/darbs_cuda.h.
 */
#ifndef DARBS_CPU_H
#define DARBS_CPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    DARBS_CPU_OK = 0,
    DARBS_CPU_INVALID_PARAMETER = 1, /* darbs::invalid_parameter   errors.hpp:10 */
    DARBS_CPU_NUMERIC_ERROR = 2,     /* darbs::numeric_error / degenerate_covariance errors.hpp:14-20 */
    DARBS_CPU_CONTRACT_VIOLATION = 4 /* darbs::contract_violation  errors.hpp:30 */
};

/* KernelFamily order of kernel.hpp:12-18. */
enum {
    DARBS_CPU_GAUSSIAN = 0,
    DARBS_CPU_HALF_COSINE = 1,
    DARBS_CPU_RAISED_COSINE = 2,
    DARBS_CPU_MODULUS_SINC = 3,
    DARBS_CPU_INVERSE_MULTIQUADRATIC = 4
};

/* KernelSpec, kernel.hpp:20-33. */
typedef struct {
    int family;
    double beta;
    double xi;
    int lobes;
    double cutoff;
    int unbounded;
} darbs_cpu_kernel;

/* Which implementation this library is: "port" or "reference". */
const char* darbs_cpu_kind(void);

/* make_kernel kernel.cpp:42-65; kernel_preset kernel.cpp:223-240. */
int darbs_cpu_make_kernel(int family, double beta, double xi, int lobes, darbs_cpu_kernel* out);
int darbs_cpu_kernel_preset(const char* name, darbs_cpu_kernel* out);
/* default_psi psi_table.hpp:20-32; returns <0 when the preset is unknown. */
double darbs_cpu_default_psi(const char* name);

/* eval kernel.cpp:127-164 over n samples. */
int darbs_cpu_eval(const darbs_cpu_kernel* k, int n, const double* dm2, double* weight,
                   double* dweight_ddm2);

/* conic_and_radius geometry.cpp:50-64.  cov2 = (a, b, c) per item. Returns
 * NUMERIC_ERROR at the first non-PD covariance (outputs up to there are valid). */
int darbs_cpu_conic_and_radius(const darbs_cpu_kernel* k, int n, const double* cov2,
                               double* conic, double* radius, double* lambda12);

/* The reference's random_scene fixture (benchmarks/bench.cpp:20-46), with the
 * draw order fixed as bench.cpp writes it: a, c, corr, mu.x, mu.y, depth,
 * opacity, r, g, b per splat from std::mt19937_64(seed) through
 * std::uniform_real_distribution<double>.  If round_f32 != 0 every field is
 * rounded to float32 (conic and radius are computed from the rounded cov2 and
 * then rounded themselves) so the GPU and the oracle consume identical values
 * (SURVEY.md §8c "parity input rule"). */
int darbs_cpu_random_scene(const darbs_cpu_kernel* k, int count, int width, int height,
                           uint64_t seed, int round_f32, double* mu2, double* cov2,
                           double* conic, double* radius, double* depth, double* opacity,
                           double* rgb);

/* Uniform(-1,1) upstream image gradient from std::mt19937_64(seed)
 * (tests/acceptance.cpp:266-270), optionally rounded to float32. */
void darbs_cpu_random_image_grad(int width, int height, uint64_t seed, int round_f32,
                                 double* grad_image);

/* bin_splats rasterizer.cpp:25-53.  tile_offsets has tiles_x*tiles_y+1 entries
 * (CSR); point_list receives up to capacity entries; depth_order (n entries,
 * may be NULL) receives the stable depth order.  Returns the total number of
 * tile entries K (even when K > capacity, in which case nothing is written to
 * point_list) or a negative status. */
int64_t darbs_cpu_bin(int n, const double* mu2, const double* conic, const double* radius,
                      const double* depth, int width, int height, int64_t* tile_offsets,
                      int32_t* point_list, int64_t capacity, int32_t* depth_order);

/* forward rasterizer.cpp:55-112.  Returns an opaque handle holding the
 * BlendAux (bins, t_final, processed, contributors) for the matching backward,
 * or NULL on error.  Output pointers may be NULL. */
void* darbs_cpu_forward(const darbs_cpu_kernel* k, int n, const double* mu2, const double* conic,
                        const double* radius, const double* depth, const double* opacity,
                        const double* rgb, int width, int height, const double* background,
                        int threads, double* image, double* t_final, int32_t* processed,
                        int32_t* contributors, int32_t* skipped_nonfinite);
void darbs_cpu_forward_free(void* handle);

/* oracle_forward rasterizer.cpp:114-145 (brute force, no tiles). */
int darbs_cpu_oracle_forward(const darbs_cpu_kernel* k, int n, const double* mu2,
                             const double* conic, const double* radius, const double* depth,
                             const double* opacity, const double* rgb, int width, int height,
                             const double* background, double* image);

/* backward rasterizer.cpp:147-234.  grads = 9 per splat in SplatGrads order
 * (rasterizer.hpp:53-60): d_color[3], d_opacity, d_conic_a, d_conic_b,
 * d_conic_c, d_mu2[2].  Returns CONTRACT_VIOLATION when the gradient image
 * size or splat count does not match the handle (rasterizer.cpp:151-154). */
int darbs_cpu_backward(void* handle, const darbs_cpu_kernel* k, int grad_width, int grad_height,
                       const double* grad_image, int n, const double* mu2, const double* conic,
                       const double* opacity, const double* rgb, int threads, double* grads);

/* realize fit3d.cpp:17-25: 14 raw parameters -> Primitive3D fields
 * (mu3, scale3, quat wxyz, opacity, rgb3), 14 doubles per primitive. */
void darbs_cpu_realize(int n, const double* raw, double* prims);

/* project_primitive geometry.cpp:66-87 for n primitives (realized layout).
 * camera = fx fy cx cy width height + 16 row-major world-to-camera entries
 * (scene_io.hpp:16-19).  valid[i] = 0 when near-plane culled.  Returns
 * INVALID_PARAMETER (scale<=0, psi<=0) or NUMERIC_ERROR (non-PD) like the
 * reference's exceptions. */
int darbs_cpu_project(const darbs_cpu_kernel* k, double psi, double dilation, int n,
                      const double* prims, const double* camera, int32_t* valid, double* mu2,
                      double* cov2, double* conic, double* radius, double* depth);

/* backward_projection geometry.cpp:111-168. grad_cov2 = (xx, xy, yx, yy). */
void darbs_cpu_backward_projection(double psi, int n, const double* grad_cov2,
                                   const double* grad_mu2, const double* prims,
                                   const double* camera, double* d_mu, double* d_scale,
                                   double* d_rot);

/* The per-view gradient chain of fit_scene's evaluate, fit3d.cpp:134-159:
 * conic grads -> cov2 grads (-C G C), backward_projection, reparametrisation,
 * "+=" into param_grads[14 * owner[k]].  splat_* arrays have m entries
 * (compacted visible splats), owner maps them to primitives. */
void darbs_cpu_param_grads(double psi, int m, const int32_t* owner, const double* splat_grads,
                           const double* conic, const double* opacity, const double* rgb,
                           const double* prims, const double* camera, double* param_grads);

/* loss_total loss.cpp:173-230: L = (1 - lambda) L1 + lambda (1 - SSIM)/2 with its analytic gradient
 * with respect to `rendered` (3*w*h, row-major RGB interleaved, like the images).  out[0..2] =
 * total, l1, dssim.  grad may be NULL. */
int darbs_cpu_loss_total(int width, int height, const double* rendered, const double* target,
                         double lambda, double out[3], double* grad);
/* ssim loss.cpp:142-171: mean SSIM over pixels and channels. */
int darbs_cpu_ssim(int width, int height, const double* a, const double* b, double* out);
/* The reference's random_image fixture (tests/test_loss.cpp:13-19): U[0,1) per value from
 * std::mt19937_64(seed), optionally rounded to float32. */
void darbs_cpu_random_image(int width, int height, uint64_t seed, int round_f32, double* rgb);

/* adam_step optim.hpp:24-39 (t is 1-based). */
int darbs_cpu_adam_step(int64_t dim, double* params, const double* grads, double* m, double* v,
                        const double* lrs, int t);

#ifdef __cplusplus
}
#endif
#endif /* DARBS_CPU_H */
