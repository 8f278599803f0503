/*
 * darbs_cuda.h — C ABI of the B200-native DARBF splatting rasterizer.
 *
 * This is the drop-in boundary for the reference's rasterizer hot path
 * (arxiv/paper_2501_12369, proj/core).  The reference has no FFI of its own:
 * its interface for this path is a handful of C++ free functions in namespace
 * darbs.  Each entry point below names the reference interface it replaces
 * (paths relative to the reference's proj/core/).  The C++ mirror of those
 * functions, with the reference's own signatures, lives in
 * paper_2501_12369_b200/host/darbs_b200.hpp and only calls this ABI.
 *
 * Conventions
 *  - plain pointers and sizes; no C++ or torch types.
 *  - every array argument of one call lives in ONE memory space, named by the
 *    `space` argument: DARBS_HOST (the library stages through its own device
 *    workspace and copies results back before returning) or DARBS_DEVICE
 *    (pointers are device pointers on the context's GPU; the call is
 *    asynchronous on the context's stream unless stated otherwise).
 *  - element type is float32 on the wire (the reference is float64; see
 *    DESIGN.md "precision policy").  Images are row-major, RGB interleaved
 *    (include/darbs/image.hpp:9-20).  Splats are structure-of-arrays.
 *  - every function returns a darbs_status; the reference's exceptions map to
 *    status codes as listed at the enum.  darbs_cuda_last_error() gives the
 *    message of the last failure on the context.
 *  - a context belongs to one host thread and one GPU; calls on it are
 *    serialised on its stream.
 *  - there is no CPU fallback: if no CUDA device is usable, create fails.
 */
#ifndef DARBS_CUDA_H
#define DARBS_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(_WIN32)
#define DARBS_API
#else
#define DARBS_API __attribute__((visibility("default")))
#endif

/* include/darbs/errors.hpp:10-36 and the CLI's exit-code mapping tools/main.cpp:487-499 */
typedef enum {
    DARBS_OK = 0,
    DARBS_INVALID_PARAMETER = 1,  /* darbs::invalid_parameter */
    DARBS_NUMERIC_ERROR = 2,      /* darbs::numeric_error, darbs::degenerate_covariance */
    DARBS_IO_ERROR = 3,           /* darbs::io_error (unused on this path) */
    DARBS_CONTRACT_VIOLATION = 4, /* darbs::contract_violation */
    DARBS_CUDA_ERROR = 5          /* CUDA runtime failure (no reference analogue) */
} darbs_status;

typedef enum { DARBS_HOST = 0, DARBS_DEVICE = 1 } darbs_space;

/* include/darbs/kernel.hpp:12-18 */
typedef enum {
    DARBS_GAUSSIAN = 0,
    DARBS_HALF_COSINE = 1,
    DARBS_RAISED_COSINE = 2,
    DARBS_MODULUS_SINC = 3,
    DARBS_INVERSE_MULTIQUADRATIC = 4
} darbs_family;

/* KernelSpec, include/darbs/kernel.hpp:20-33 */
typedef struct {
    int32_t family;
    double beta;
    double xi;
    int32_t lobes;
    double cutoff;
    int32_t unbounded;
} darbs_kernel_spec;

/* rasterizer constants, include/darbs/rasterizer.hpp:11-14 */
#define DARBS_TILE_SIZE 16
#define DARBS_ALPHA_CLAMP 0.99
#define DARBS_ALPHA_SKIP (1.0 / 255.0)
#define DARBS_TRANSMITTANCE_FLOOR 1e-4
/* include/darbs/geometry.hpp:55-56 */
#define DARBS_NEAR_PLANE 0.01
#define DARBS_DILATION 0.3
/* fit3d.cpp:15 — mu(3) log_scale(3) quat wxyz(4) logit_opacity logit_rgb(3) */
#define DARBS_PARAMS_PER_PRIMITIVE 14
/* SplatGrads, include/darbs/rasterizer.hpp:53-60: d_color[3] d_opacity d_conic_a d_conic_b d_conic_c d_mu2[2] */
#define DARBS_GRADS_PER_SPLAT 9
/* camera block, include/darbs/scene_io.hpp:16-19: fx fy cx cy width height + 16 row-major world-to-camera */
#define DARBS_CAMERA_DOUBLES 22

typedef struct darbs_cuda_ctx darbs_cuda_ctx;

/* ---- library / context ---------------------------------------------------- */

DARBS_API const char* darbs_cuda_version(void);

/* Creates a context on CUDA device `device` with its own non-blocking stream. */
DARBS_API darbs_status darbs_cuda_create(int device, darbs_cuda_ctx** out_ctx);
DARBS_API void darbs_cuda_destroy(darbs_cuda_ctx* ctx);
/* Message of the last non-OK status on this context ("" if none); ctx may be
 * NULL for create failures. */
DARBS_API const char* darbs_cuda_last_error(const darbs_cuda_ctx* ctx);
/* Use an externally owned cudaStream_t (e.g. torch's current stream) for all
 * subsequent work; NULL restores the context's own stream.  To run on the legacy
 * default stream pass cudaStreamLegacy ((void*)1), not NULL.  Switching drains the stream that is
 * left; binding the stream the context already runs on is free (and legal while that stream is
 * capturing a CUDA graph). */
DARBS_API darbs_status darbs_cuda_set_stream(darbs_cuda_ctx* ctx, void* cuda_stream);
DARBS_API darbs_status darbs_cuda_synchronize(darbs_cuda_ctx* ctx);
/* Number of kernels this library has launched on the context since creation
 * (all of them its own: no library kernel is called). */
DARBS_API int64_t darbs_cuda_launch_count(const darbs_cuda_ctx* ctx);
/* 1: decisions that fall inside the FP32 guard band of a threshold are re-taken
 * in FP64 exactly as the reference takes them (default).  0: pure FP32. */
DARBS_API darbs_status darbs_cuda_set_exact_decisions(darbs_cuda_ctx* ctx, int enabled);
/* Deterministic reduction (default 0).  The reference's backward writes per-tile gradient buffers
 * and reduces them in a fixed order, so its results do not depend on the thread count
 * (src/rasterizer.cpp:159-165, :219-232; tests/test_rasterizer.cpp:260-273).  With 1 the render
 * backward accumulates the per-block partial gradients, and the loss kernels their partial sums,
 * as 64-bit FIXED-POINT integers (2^-36 resolution, range +-1.3e8): integer addition is
 * associative, so the result is bitwise independent of the order in which blocks arrive and a
 * rerun is bitwise identical.  0: float32 vector reductions (faster; equal up to summation order). */
DARBS_API darbs_status darbs_cuda_set_deterministic(darbs_cuda_ctx* ctx, int enabled);
/* evaluate_view / train_step normally wait (an event, not the stream) for ONE number of a view,
 * K = the total of tile entries, to size the entry buffers.  A caller that knows a bound — a
 * training loop whose previous iterations saw K_prev can pass 1.25 K_prev — sets it here
 * (entries > 0) and the wait disappears: buffers and grids are sized by the capacity, the kernels
 * take K from the device, and an iteration can be queued without any host synchronisation
 * (CUDA-graph capturable: darbs_cuda_evaluate_view with DARBS_DEVICE arrays on a capturing stream
 * records the whole view; such a view reports neither loss nor status - loss_out must be NULL and
 * nothing is queued for darbs_cuda_pop_loss - so check K <= capacity with an eager view now and
 * then; darbs_cuda_adam_step takes its bias correction by value and is launched outside the graph;
 * tests/test_gpu_geometry.py::test_a_view_is_capturable_in_a_cuda_graph, bench.py's device-resident
 * arm).  A view with K > capacity is TRUNCATED safely (no write leaves the
 * buffers) and reported as DARBS_CONTRACT_VIOLATION by the call that collects its loss
 * (darbs_cuda_pop_loss, or evaluate_view / train_step with loss_out).  0 restores the wait.
 * Heuristics that look at K (the cull segment) take the capacity to be 1.25 x the expected K.
 * Only the fused training path honours it; darbs_cuda_forward / darbs_cuda_bin always wait. */
DARBS_API darbs_status darbs_cuda_set_entry_capacity(darbs_cuda_ctx* ctx, int64_t entries);
/* Tuning knob without a reference analogue.  The cull kernel tests only the first `entries` list
 * entries of every tile against its eight 8x4 pixel blocks; a block whose pixels are still live
 * behind them culls on by itself inside the forward kernel.  Results do not depend on the value
 * (the per-pixel walk is the reference's, rasterizer.cpp:85-107); 0 (default) picks per family. */
DARBS_API darbs_status darbs_cuda_set_cull_segment(darbs_cuda_ctx* ctx, int entries);

/* ---- device memory ----------------------------------------------------------
 * For callers without a CUDA toolchain of their own (the C++ mirror's fit_scene keeps the raw
 * parameters, Adam state and target images resident on the GPU; the reference keeps its
 * std::vectors in host memory, so these have no reference analogue).  Pointers returned by
 * device_alloc are DARBS_DEVICE pointers for every entry point of this header.  upload is
 * stream-ordered (the host buffer may be reused on return); download synchronises. */
DARBS_API darbs_status darbs_cuda_device_alloc(darbs_cuda_ctx* ctx, uint64_t bytes, void** out_ptr);
DARBS_API darbs_status darbs_cuda_device_free(darbs_cuda_ctx* ctx, void* ptr);
DARBS_API darbs_status darbs_cuda_upload(darbs_cuda_ctx* ctx, void* dst_device, const void* src_host,
                                         uint64_t bytes);
DARBS_API darbs_status darbs_cuda_download(darbs_cuda_ctx* ctx, void* dst_host, const void* src_device,
                                           uint64_t bytes);
DARBS_API darbs_status darbs_cuda_device_zero(darbs_cuda_ctx* ctx, void* ptr, uint64_t bytes);

/* ---- kernel family ---------------------------------------------------------- */

/* make_kernel, src/kernel.cpp:42-65 (host-side; validates and fills cutoff). */
DARBS_API darbs_status darbs_cuda_make_kernel(int family, double beta, double xi, int lobes,
                                              darbs_kernel_spec* out);
/* kernel_preset, src/kernel.cpp:223-240: "gaussian", "half-cosine-sq",
 * "raised-cosine", "mod-sinc", "inv-multiquadratic". */
DARBS_API darbs_status darbs_cuda_kernel_preset(const char* name, darbs_kernel_spec* out);
/* default_psi, include/darbs/psi_table.hpp:20-32; negative when unknown. */
DARBS_API double darbs_cuda_default_psi(const char* name);
/* eval, src/kernel.cpp:127-164, on the device functors the render kernels use
 * (FP32 fast path; `exact` != 0 evaluates the FP64 path instead). */
DARBS_API darbs_status darbs_cuda_eval(darbs_cuda_ctx* ctx, const darbs_kernel_spec* kernel,
                                       int64_t n, const float* dm2, float* weight,
                                       float* dweight_ddm2, int exact, darbs_space space);

/* ---- rasterizer ------------------------------------------------------------- */

/* bin_splats, src/rasterizer.cpp:25-53 (TileBins, include/darbs/rasterizer.hpp:16-20).
 * Outputs (each may be NULL): num_entries (host int64, always host);
 * tile_ranges [2*tiles] = (begin, end) into point_list per tile, row-major tiles;
 * point_list [K] = splat indices, depth-ascending per tile, ties by index;
 * sort_keys  [K] = (tile_id << 32) | depth-order rank of the entry's splat;
 * depth_order[n] = splat indices in stable depth order.  `capacity` bounds the
 * K-sized outputs; if K > capacity they are not written and the call still
 * returns DARBS_OK with *num_entries = K. */
DARBS_API darbs_status darbs_cuda_bin(darbs_cuda_ctx* ctx, int64_t n, const float* mu2,
                                      const float* conic, const float* radius, const float* depth,
                                      int width, int height, int64_t* num_entries,
                                      int32_t* tile_ranges, int32_t* point_list,
                                      uint64_t* sort_keys, int32_t* depth_order, int64_t capacity,
                                      darbs_space space);

/* forward, src/rasterizer.cpp:55-112 (ForwardResult / BlendAux,
 * include/darbs/rasterizer.hpp:27-46).  mu2[2n], conic[3n] (a,b,c), radius[n],
 * depth[n], opacity[n], rgb[3n].  Outputs (each may be NULL): image[3*w*h],
 * t_final[w*h], processed[w*h], contributors[w*h], skipped_nonfinite (host int).
 * The bins and per-pixel aux stay resident in the context for the matching
 * darbs_cuda_backward, replacing the BlendAux value the reference hands back.
 * `threads` of the reference signature has no meaning here and is omitted. */
DARBS_API darbs_status darbs_cuda_forward(darbs_cuda_ctx* ctx, const darbs_kernel_spec* kernel,
                                          int64_t n, const float* mu2, const float* conic,
                                          const float* radius, const float* depth,
                                          const float* opacity, const float* rgb, int width,
                                          int height, const float background[3], float* image,
                                          float* t_final, int32_t* processed,
                                          int32_t* contributors, int32_t* skipped_nonfinite,
                                          darbs_space space);

/* backward, src/rasterizer.cpp:147-234.  grads[9n] in SplatGrads order.  Returns
 * DARBS_CONTRACT_VIOLATION when (grad_width, grad_height, n) do not match the
 * last forward on this context (rasterizer.cpp:151-154), or when `kernel` is not the
 * kernel that forward ran with.  The resident aux (bins, per-block survivor streams,
 * t_final, processed) already holds everything of the splats the backward needs, so the
 * four splat arrays are part of the signature only to mirror the reference's and are NOT
 * read: the gradients are those of the splats the matching forward call consumed
 * (the reference, handed different splats with an old aux, would mix the two; that use is
 * outside its contract as well, rasterizer.hpp:27-37).  Pass them as NULL. */
DARBS_API darbs_status darbs_cuda_backward(darbs_cuda_ctx* ctx, const darbs_kernel_spec* kernel,
                                           int grad_width, int grad_height,
                                           const float* grad_image, int64_t n, const float* mu2,
                                           const float* conic, const float* opacity,
                                           const float* rgb, float* grads, darbs_space space);

/* ---- geometry (per-primitive preprocess) ---------------------------------- */

/* realize, src/fit3d.cpp:17-25: raw[14n] -> prims[14n] (mu, scale, quat wxyz, opacity, rgb). */
DARBS_API darbs_status darbs_cuda_realize(darbs_cuda_ctx* ctx, int64_t n, const float* raw,
                                          float* prims, darbs_space space);

/* project_primitive, src/geometry.cpp:66-87, for n realized primitives.
 * camera: 22 doubles, always host.  valid[i] = 0 when near-plane culled.
 * cov2[3n] = (xx, xy, yy).  Status: INVALID_PARAMETER (scale <= 0, psi <= 0),
 * NUMERIC_ERROR (covariance not positive definite), as the reference throws. */
DARBS_API darbs_status darbs_cuda_project(darbs_cuda_ctx* ctx, const darbs_kernel_spec* kernel,
                                          double psi, double dilation, int64_t n,
                                          const float* prims, const double* camera,
                                          int32_t* valid, float* mu2, float* cov2, float* conic,
                                          float* radius, float* depth, darbs_space space);

/* backward_projection, src/geometry.cpp:111-168. grad_cov2[4n] = (xx,xy,yx,yy),
 * grad_mu2[2n]; outputs d_mu[3n], d_scale[3n], d_rot[4n] (w,x,y,z). */
DARBS_API darbs_status darbs_cuda_backward_projection(darbs_cuda_ctx* ctx, double psi, int64_t n,
                                                      const float* grad_cov2,
                                                      const float* grad_mu2, const float* prims,
                                                      const double* camera, float* d_mu,
                                                      float* d_scale, float* d_rot,
                                                      darbs_space space);

/* ---- training step (fit_scene's evaluate + adam_step) ----------------------- */

/* One view of fit_scene's evaluate lambda, src/fit3d.cpp:108-159:
 *   realize -> project_primitive (near-plane cull) -> forward -> loss ->
 *   backward -> conic-grad -> cov2-grad -> backward_projection ->
 *   reparametrisation -> param_grads[14n] += .
 * raw_params[14n] and param_grads[14n] follow `param_space`; target, grad_image
 * and image_out follow `image_space` (a training loop keeps the parameters on the
 * device and feeds each view's target image from the host).  Exactly one of
 * `target` / `grad_image` is non-NULL:
 *   target     [3wh]: loss_total(image, target, lambda) (src/loss.cpp:173-230)
 *                     drives the backward; *loss_out receives total, l1, dssim, mse.
 *   grad_image [3wh]: used as dL/dimage directly (loss_out gets zeros).
 * lambda in [0, 1] (fit_common.hpp:16 defaults to 0.2); other values return
 * DARBS_INVALID_PARAMETER.  image_out (may be NULL) receives the rendered view.
 * background: fit_scene uses (0,0,0) (fit3d.cpp:52).
 * Returns NUMERIC_ERROR when every primitive is culled (fit3d.cpp:117-119) or
 * the loss is not finite (fit3d.cpp:123-125); those checks need the results on the
 * host: with loss_out they synchronise here, with loss_out == NULL they are
 * reported by darbs_cuda_pop_loss. */
DARBS_API darbs_status darbs_cuda_evaluate_view(darbs_cuda_ctx* ctx,
                                                const darbs_kernel_spec* kernel, double psi,
                                                int64_t n, const float* raw_params,
                                                const double* camera, const float background[3],
                                                const float* target, double lambda,
                                                const float* grad_image, float* param_grads,
                                                float* image_out, double loss_out[4],
                                                darbs_space param_space,
                                                darbs_space image_space);

/* param_grads of darbs_cuda_evaluate_view: 1 (default) adds the view's gradients to what the
 * array holds (fit3d.cpp:148-158); 0 makes the NEXT evaluate_view overwrite it, which is the
 * reference's std::fill(grads, 0) (fit3d.cpp:107) followed by the first view's "+=" without the
 * pass over the array that zeroes it.  The setting returns to 1 after that call. */
DARBS_API darbs_status darbs_cuda_set_accumulate(darbs_cuda_ctx* ctx, int accumulate);

/* Starts the upload of a view's target image (host memory, pinned for a truly asynchronous copy;
 * count = 3*w*h floats) ahead of the darbs_cuda_evaluate_view call that will pass the same
 * pointer as `target` with image_space = DARBS_HOST.  The transfer is queued on the context's
 * copy stream behind the cull kernel of the last view queued, i.e. it runs under that view's
 * render kernels.  Two uploads may be outstanding; the image must not change until its
 * evaluate_view has been queued, and a staged image is recognised by its host POINTER alone: do not
 * free the buffer and reuse its address for another image between the two calls.  A second prefetch
 * into a slot waits for the loss kernels that read the slot's previous image.  Without a prefetch
 * evaluate_view uploads the image itself. */
DARBS_API darbs_status darbs_cuda_prefetch_target(darbs_cuda_ctx* ctx, const float* host_image,
                                                  int64_t count);

/* Collects (total, l1, dssim, mse) and the status of the OLDEST darbs_cuda_evaluate_view that was
 * called with loss_out == NULL (fit3d.cpp:117-125, :161-165), waiting only for that view's
 * results.  Up to 4 views may be pending (older ones are forgotten); a training loop pops the loss of iteration i after it
 * has queued iteration i + 1, so the GPU never idles on the read-back.  Passing loss_out to
 * evaluate_view is the synchronous form (it drains everything pending). */
DARBS_API darbs_status darbs_cuda_pop_loss(darbs_cuda_ctx* ctx, double loss_out[4]);

/* loss_total, src/loss.cpp:173-230 (LossResult, include/darbs/loss.hpp:7-12):
 * L = (1 - lambda) L1 + lambda (1 - SSIM)/2 with the 11x11 sigma-1.5 window and mirror padding,
 * and its analytic gradient with respect to `rendered`.  rendered, target, grad_image: [3wh],
 * row-major RGB interleaved.  loss_out (host, may be NULL; synchronises when given) receives
 * total, l1, dssim, mse; grad_image may be NULL (values only).  The reference throws
 * invalid_parameter on a dimension mismatch (loss.cpp:174-176); here both images share the one
 * (width, height) of the call. */
DARBS_API darbs_status darbs_cuda_loss_total(darbs_cuda_ctx* ctx, int width, int height,
                                             const float* rendered, const float* target,
                                             double lambda, double loss_out[4], float* grad_image,
                                             darbs_space space);

/* adam_step, include/darbs/optim.hpp:24-39 (beta1 .9, beta2 .999, eps 1e-15,
 * per-parameter learning rates, t is 1-based). */
DARBS_API darbs_status darbs_cuda_adam_step(darbs_cuda_ctx* ctx, int64_t dim, float* params,
                                            const float* grads, float* m, float* v,
                                            const float* lrs, int t, darbs_space space);

/* ---- multi-GPU: view-parallel training iteration ------------------------------
 * fit_scene's iteration, src/fit3d.cpp:104-184, with the view loop sharded over the ranks of one
 * node (one process and one context per GPU; view v belongs to rank v mod world).
 * Every rank keeps a replica of params / m / v; the only exchange on the path is ONE all-reduce
 * (sum, no 1/V scaling: the reference sums, fit3d.cpp:148-158) of the 14 n float32 gradient
 * buffer per iteration, over NCCL (NVLink / NVSwitch), issued on its own stream in pieces so
 * that Adam updates a piece while the next is still being reduced.  NCCL is bound at run time
 * (dlopen libnccl.so.2; the environment variable DARBS_NCCL_LIB overrides the name), so the
 * single-GPU entry points have no dependency on it.  Without a communicator (or world == 1)
 * darbs_cuda_train_step is the plain single-GPU iteration. */
typedef struct { char bytes[128]; } darbs_comm_id;   /* ncclUniqueId */
/* Rank 0 makes the id and hands it to the other ranks by any means (file, socket, MPI). */
DARBS_API darbs_status darbs_cuda_comm_unique_id(darbs_comm_id* out);
/* Collective over all ranks (ncclCommInitRank).  Replaces an existing communicator. */
DARBS_API darbs_status darbs_cuda_comm_init(darbs_cuda_ctx* ctx, const darbs_comm_id* id, int rank,
                                            int world);
DARBS_API darbs_status darbs_cuda_comm_destroy(darbs_cuda_ctx* ctx);
/* The exchange and the update alone (fit3d.cpp:148-158's "+=" across ranks, then optim.hpp:24-39):
 * grads[dim] (DARBS_DEVICE, already holding this rank's views) is all-reduced over the context's
 * communicator in pieces on a side stream and Adam step t follows piece by piece.  For callers
 * that evaluate their views themselves (e.g. with host-resident target images). */
DARBS_API darbs_status darbs_cuda_allreduce_adam_step(darbs_cuda_ctx* ctx, int64_t dim, float* params,
                                                      float* grads, float* m, float* v,
                                                      const float* lrs, int t);
/* One iteration.  All arrays are DARBS_DEVICE: params, grads, m, v, lrs [14 n]; cameras
 * [n_local_views][22]; targets[n_local_views] device pointers to [3wh] images of the cameras'
 * sizes.  The rank's local views are evaluated (the first overwrites `grads`, fit3d.cpp:107),
 * `grads` is all-reduced, Adam step `t` (1-based) is applied.  loss_out (may be NULL) receives
 * the mean over all n_views_total views of (total, l1, dssim, mse) (fit3d.cpp:161-165; a second
 * all-reduce of four doubles, which synchronises).  Errors of a view (all primitives culled,
 * non-finite loss) are reported after the iteration has been queued, like darbs_cuda_pop_loss. */
DARBS_API darbs_status darbs_cuda_train_step(darbs_cuda_ctx* ctx, const darbs_kernel_spec* kernel,
                                             double psi, int64_t n, float* params, float* grads,
                                             float* m, float* v, const float* lrs,
                                             int n_local_views, const double* cameras,
                                             const float* const* targets, double lambda,
                                             const float background[3], int t, int n_views_total,
                                             double loss_out[4]);

/* ---- instrumentation ---------------------------------------------------------- */

/* Device time in milliseconds of the stages of the last forward / backward /
 * evaluate_view on this context, measured with CUDA events on the context's
 * stream (synchronises).  out[0..7] = preprocess, binning (sort and tile ranges),
 * render_fwd, loss, render_bwd, preprocess_bwd, adam, cull (record packing and
 * the per-block survivor streams).  Recording is off by default. */
DARBS_API darbs_status darbs_cuda_set_stage_timing(darbs_cuda_ctx* ctx, int enabled);
DARBS_API darbs_status darbs_cuda_stage_times(darbs_cuda_ctx* ctx, double out_ms[8]);
/* Work counters of the last forward: out[0] = K tile entries, out[1] = sum of
 * processed (visits), out[2] = sum of contributors, out[3] = (8x4 pixel block,
 * entry) pairs that survived the block-level cull, out[4] = FP64 guard-band
 * re-decisions, out[5] = pixels flagged near the transmittance floor, out[6] =
 * (block, entry) pairs the forward composited before its early exits.
 * Synchronises. */
DARBS_API darbs_status darbs_cuda_work_counters(darbs_cuda_ctx* ctx, int64_t out[8]);

/* Register-only micro-benchmarks of the two pipes that bound the render kernels,
 * run on the context's GPU (a few milliseconds): out[0] = FP32 FMA instructions
 * per second with register operands (x2 = FLOP/s), out[1] = MUFU (ex2.approx)
 * operations per second, out[2] = SM clock in MHz seen by the FMA loop (clock64
 * span / event time), out[3] = number of SMs, out[4] = FP32 FMA instructions per
 * second in the immediate-operand form, out[5] = packed FP32 FMA instructions
 * (fma.rn.f32x2, two FMAs per lane) per second. */
DARBS_API darbs_status darbs_cuda_microbench(darbs_cuda_ctx* ctx, double out[8]);

#ifdef __cplusplus
}
#endif
#endif /* DARBS_CUDA_H */
