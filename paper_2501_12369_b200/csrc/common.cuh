// common.cuh — shared declarations of the sm_100a implementation behind
// include/darbs_cuda.h: context, grow-only device workspace, kernel-family
// parameters and the packed splat record the render kernels consume.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "darbs_cuda.h"

namespace darbs_b200 {

// ---------------------------------------------------------------- families
// Compile-time specialisations of the DARBF family (kernel.cpp:73-104 /
// :127-164).  The four presets of the paper get a closed form on the scaled
// squared distance m = scale * dm2 (and so does the reference's fifth preset, mod-sinc);
// every other (family, beta, lobes) combination runs through FAM_GENERIC.
enum : int {
    FAM_GAUSS2 = 0,   // Gaussian, beta = 2:            w = exp(-dm2/xi)
    FAM_HCOS2 = 1,    // half-cosine, beta = 2:         w = cos(dm2/xi)
    FAM_RCOS1 = 2,    // raised-cosine, beta = 1, 1 lobe: w = .5 + .5 cos(sqrt(dm2)/xi)
    FAM_IMQ = 3,      // inverse multiquadric:          w = 1/sqrt(dm2/xi + 1)
    FAM_MSINC1 = 4,   // modulus sinc, beta = 1, 1 lobe: w = sin(u)/u, u = sqrt(dm2)/xi in [0, pi]
    FAM_GENERIC = 5   // anything else (multi-lobe, other beta)
};

struct KParams {
    int fam;        // FAM_*
    int family;     // darbs_family
    int lobes;
    int unbounded;
    int exact;      // FP64 re-decision inside the guard band
    float beta, xi, cutoff;
    float scale;    // m = scale * dm2 (>0)
    float band;     // guard band half-width, in m units
    double beta_d, xi_d, cutoff_d;
};

// Packed per-splat record, 4 x float4 = 64 B, 64-B aligned (two 32-B sectors
// per gather for the three hot vectors):
//   v0 = { mu.x, mu.y, A = scale*a, C = scale*c }   (A, C) adjacent: one packed multiply with (dx^2, dy^2)
//   v1 = { B = scale*2b, opacity, thr_m, -b/c }     thr_m: see family_threshold()
//   v2 = { r, g, b, -b/a }                          v1.w, v2.w: block-cull helpers
//   v3 = { a, b, c, 0 }                          unscaled conic for the FP64 path
static constexpr int kRecVecs = 4;

// Fixed-point accumulation of the deterministic mode: value * 2^36 rounded to int64, added with
// integer atomics (associative: the sum does not depend on the order of arrival).
static constexpr double kFixedScale = 68719476736.0;  // 2^36

// ---------------------------------------------------------------- workspace
struct DeviceBuffer {
    void* ptr = nullptr;
    size_t bytes = 0;
};

struct Counters {  // device-side, 8 x u64
    unsigned long long v[8];
};

// One evaluate_view whose loss has not been collected yet: the device -> host copy of its status
// flags and loss sums lands in `host` (pinned) when `done` fires.
static constexpr int kLossRing = 4;
struct LossSlot {
    void* host = nullptr;
    cudaEvent_t done = nullptr;
    double count = 0.0;   // number of image values, 0 when the view had no target
    double lambda = 0.0;
    bool fixed_point = false;  // the three sums are int64 fixed point (deterministic mode)
};

struct StageTimer {
    cudaEvent_t ev[16];
    bool created = false;
};

}  // namespace darbs_b200

struct darbs_cuda_ctx {
    int device = 0;
    int sm_count = 148;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    // host -> device uploads that a call does not need until late (the target image of
    // evaluate_view) run on their own stream, fenced by these two events
    cudaStream_t copy_stream = nullptr;
    cudaStream_t aux_stream = nullptr;                       // the tile ordering runs here, under the cull kernel
    cudaEvent_t ranges_ready = nullptr, order_ready = nullptr;
    bool tile_order_pending = false;                         // the stream has not yet waited for order_ready
    bool tile_order_wanted = false;                          // a forward follows this binning
    cudaEvent_t copy_begin = nullptr, copy_done = nullptr;
    std::string last_error;
    int64_t launches = 0;
    int exact = 1;
    int timing = 0;
    int64_t entry_capacity = 0;  // > 0: evaluate_view does not wait for K (darbs_cuda_set_entry_capacity)
    int cull_segment = 0;   // entries of a tile's list the cull kernel covers (0: per family, render.cu cull_segment)
    int deterministic = 0;  // fixed-point accumulation of gradients and loss sums (darbs_cuda_set_deterministic)
    int accumulate = 1;  // evaluate_view adds to param_grads (0: the next call overwrites)
    double stage_ms[8] = {0, 0, 0, 0, 0, 0, 0, 0};

    // grow-only device workspace
    darbs_b200::DeviceBuffer recs;         // n * 64 B packed records
    darbs_b200::DeviceBuffer rects;        // n * uint2 (packed tile rect, tiles touched)
    darbs_b200::DeviceBuffer depth_keys;   // 2 * n u32 (double buffer)
    darbs_b200::DeviceBuffer order;        // 2 * n u32 (double buffer)
    darbs_b200::DeviceBuffer tile_keys;    // 2 * K u32
    darbs_b200::DeviceBuffer tile_vals;    // 2 * K u32
    darbs_b200::DeviceBuffer ranges;       // tiles * int2
    darbs_b200::DeviceBuffer streams;      // 8 (K + 32 tiles) x 48 B: per-block survivor streams (render.cu)
    darbs_b200::DeviceBuffer stream_count; // 2 x 8 tiles int: entries per stream | entries the forward composited
    darbs_b200::DeviceBuffer sort_ws;      // tickets, digit histograms and status words of the sorts (binning.cu)
    darbs_b200::DeviceBuffer tile_status;  // status words of the tile sort's passes (sized by K)
    darbs_b200::DeviceBuffer tile_order;   // tiles int: tile indices, longest list first (the render kernels' CTA order)
    bool tile_order_valid = false;         // set by the tile sort of the current forward
    int tile_order_lpt = 1;                // 0: CTAs take the tiles in raster order
    darbs_b200::DeviceBuffer counters;     // Counters + scalars
    darbs_b200::DeviceBuffer t_final, processed, contributors, image;  // per-pixel aux
    darbs_b200::DeviceBuffer stage_in[8];  // staging for DARBS_HOST calls / internal SoA
    darbs_b200::DeviceBuffer stage_out[8];
    darbs_b200::DeviceBuffer valid;        // per-primitive visibility (evaluate_view)
    darbs_b200::DeviceBuffer splat_grads;  // 12n: SplatGrads rows padded to 12 floats
    darbs_b200::DeviceBuffer splat_grads_fx;  // 9n int64: the same sums in fixed point (deterministic mode)
    darbs_b200::DeviceBuffer grad_image;   // 3wh
    darbs_b200::DeviceBuffer loss_maps;    // 9wh: the three SSIM partial maps (loss.cu)
    void* pinned = nullptr;                // small pinned host scratch
    size_t pinned_bytes = 0;

    // target images uploaded ahead of the evaluate_view that uses them (darbs_cuda_prefetch_target)
    darbs_b200::DeviceBuffer target_stage[2];
    const void* target_src[2] = {nullptr, nullptr};
    cudaEvent_t target_done[2] = {nullptr, nullptr};
    cudaEvent_t target_read[2] = {nullptr, nullptr};  // recorded behind the slot's last reader (the loss kernels)
    bool target_read_pending[2] = {false, false};
    int target_next = 0;
    cudaEvent_t after_cull = nullptr;  // the last forward's long kernels start here
    cudaEvent_t k_ready = nullptr;     // binning: the entry count K has reached pinned host memory
    bool have_after_cull = false;

    darbs_b200::LossSlot loss_ring[darbs_b200::kLossRing];
    int loss_head = 0, loss_pending = 0;

    // state of the last forward (the resident BlendAux)
    bool have_forward = false;
    int fwd_family = -1, fwd_lobes = 0;  // the kernel the last forward ran with
    double fwd_beta = 0.0, fwd_xi = 0.0;
    int64_t fwd_n = 0;
    int fwd_w = 0, fwd_h = 0;
    int tiles_x = 0, tiles_y = 0;
    int64_t fwd_entries = 0;
    float fwd_bg[3] = {0, 0, 0};
    const int32_t* fwd_contrib = nullptr;  // device array the last forward wrote contributors to
    int cur_key_buf = 0;  // which half of tile_vals holds the sorted point list
    int cur_order_buf = 0;

    darbs_b200::StageTimer timer;
    void* comm = nullptr;  // darbs_b200::Comm (multigpu.cu): the NCCL communicator of darbs_cuda_comm_init
};

namespace darbs_b200 {

// ---------------------------------------------------------------- errors
darbs_status fail(darbs_cuda_ctx* ctx, darbs_status st, const std::string& msg);
darbs_status cuda_fail(darbs_cuda_ctx* ctx, cudaError_t e, const char* what);

#define DARBS_CUDA_TRY(ctx, expr)                                         \
    do {                                                                  \
        cudaError_t _e = (expr);                                          \
        if (_e != cudaSuccess) return darbs_b200::cuda_fail(ctx, _e, #expr); \
    } while (0)

#define DARBS_TRY(expr)                        \
    do {                                       \
        darbs_status _s = (expr);              \
        if (_s != DARBS_OK) return _s;         \
    } while (0)

darbs_status reserve(darbs_cuda_ctx* ctx, DeviceBuffer& buf, size_t bytes);
darbs_status reserve_pinned(darbs_cuda_ctx* ctx, size_t bytes);
darbs_status check_launch(darbs_cuda_ctx* ctx, const char* what, int launches = 1);

// host-side kernel validation shared by the ABI (kernel.cpp:42-65)
darbs_status make_kparams(darbs_cuda_ctx* ctx, const darbs_kernel_spec* spec, KParams* out);

// Where the fused preprocess leaves what binning and the render kernels need (all null when the
// stages run separately).
static constexpr int kSlotsK = 64;       // K is accumulated over this many addresses, by block index
static constexpr int kSlotsKBase = 32;   // their position in ctx->counters, in u64 units
static constexpr int kOverflowAt = 13;   // entry-capacity overflow flag (u64), inside the 40 bytes a loss slot copies

struct SplatSinks {
    float4* recs = nullptr;           // n x kRecVecs
    uint2* rects = nullptr;           // n
    unsigned* touched = nullptr;      // n
    unsigned* depth_keys = nullptr;   // n
    unsigned* order = nullptr;        // n
    unsigned long long* skipped_nonfinite = nullptr;
    unsigned long long* k_slots = nullptr;  // kSlotsK partial sums of the tile counts (K = their total)
    int tiles_x = 0, tiles_y = 0;
};

// ---------------------------------------------------------------- launchers
// render.cu
darbs_status launch_pack(darbs_cuda_ctx* ctx, const KParams& kp, int64_t n, const float* mu2,
                         const float* conic, const float* opacity, const float* rgb);
darbs_status launch_render_fwd(darbs_cuda_ctx* ctx, const KParams& kp, int width, int height,
                               const float bg[3], float* image, float* t_final,
                               int32_t* processed, int32_t* contributors);
darbs_status launch_cull(darbs_cuda_ctx* ctx, const KParams& kp);
darbs_status launch_render_bwd(darbs_cuda_ctx* ctx, const KParams& kp, int width, int height,
                               const float bg[3], const float* grad_image, const float* t_final,
                               const int32_t* processed, int64_t n);
darbs_status launch_export_grads(darbs_cuda_ctx* ctx, int64_t n, float* out);
static constexpr int kSplatGradRow = 12;  // floats per row of ctx->splat_grads
darbs_status launch_eval(darbs_cuda_ctx* ctx, const KParams& kp, int64_t n, const float* dm2,
                         float* w, float* dw, int exact);
darbs_status launch_sum_counts(darbs_cuda_ctx* ctx, int64_t px, const int32_t* processed,
                               const int32_t* contributors);

// binning.cu
darbs_status binning_begin(darbs_cuda_ctx* ctx, int64_t n, int width, int height, SplatSinks* sinks);
darbs_status run_binning(darbs_cuda_ctx* ctx, int64_t n, const float* mu2, const float* conic,
                         const float* radius, const float* depth, const int32_t* valid,
                         int width, int height, bool rects_done = false);
darbs_status export_bins(darbs_cuda_ctx* ctx, int64_t n, int32_t* tile_ranges, int32_t* point_list,
                         uint64_t* sort_keys, int32_t* depth_order);
const int32_t* point_list_ptr(const darbs_cuda_ctx* ctx);
const uint32_t* depth_order_ptr(const darbs_cuda_ctx* ctx);

// multigpu.cu
void destroy_comm(darbs_cuda_ctx* ctx);

// geometry.cu
struct CameraD {
    double fx, fy, cx, cy;
    double w[12];  // rows 0..2 of the world-to-camera transform (3x4)
    int width, height;
};
CameraD make_camera(const double* cam22);
darbs_status launch_realize(darbs_cuda_ctx* ctx, int64_t n, const float* raw, float* prims);
darbs_status launch_project(darbs_cuda_ctx* ctx, const KParams& kp, double psi, double dilation,
                            int64_t n, const float* params, bool raw, const CameraD& cam,
                            int32_t* valid, float* mu2, float* cov2, float* conic, float* radius,
                            float* depth, float* opacity, float* rgb, int* status_flags,
                            const SplatSinks* sinks = nullptr);
darbs_status launch_backward_projection(darbs_cuda_ctx* ctx, double psi, int64_t n,
                                        const float* grad_cov2, const float* grad_mu2,
                                        const float* prims, const CameraD& cam, float* d_mu,
                                        float* d_scale, float* d_rot);
darbs_status launch_param_grads(darbs_cuda_ctx* ctx, double psi, int64_t n, const float* raw,
                                const CameraD& cam, const int32_t* valid, const float* splat_grads,
                                const float* conic, float* param_grads, bool overwrite);
darbs_status launch_adam(darbs_cuda_ctx* ctx, int64_t dim, float* params, const float* grads,
                         float* m, float* v, const float* lrs, int t);
darbs_status launch_l1_loss(darbs_cuda_ctx* ctx, int64_t count, const float* image,
                            const float* target, double lambda, float* grad_image,
                            double* sums /* device: abs sum, sq sum */);

// loss.cu
darbs_status launch_loss(darbs_cuda_ctx* ctx, int width, int height, const float* image,
                         const float* target, double lambda, float* grad_image,
                         double* sums /* device, 5 doubles: abs sum, sq sum, sum of (1 - SSIM), 2 scratch */);

}  // namespace darbs_b200
