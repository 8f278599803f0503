// api.cu — the C ABI of include/darbs_cuda.h: context, workspace, host<->device
// staging, argument validation with the reference's error taxonomy, and the
// sequencing of the stage launchers (render.cu, binning.cu, geometry.cu).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <initializer_list>
#include <new>

#include "common.cuh"
#include "family.cuh"

using namespace darbs_b200;

namespace darbs_b200 {

static thread_local std::string g_create_error;

darbs_status fail(darbs_cuda_ctx* ctx, darbs_status st, const std::string& msg) {
    if (ctx)
        ctx->last_error = msg;
    else
        g_create_error = msg;
    return st;
}

darbs_status cuda_fail(darbs_cuda_ctx* ctx, cudaError_t e, const char* what) {
    return fail(ctx, DARBS_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

darbs_status reserve(darbs_cuda_ctx* ctx, DeviceBuffer& buf, size_t bytes) {
    bytes = (bytes + 255) & ~(size_t)255;
    if (bytes <= buf.bytes) return DARBS_OK;
    // grow-only, with head-room so that a slowly growing K does not reallocate every frame
    size_t want = bytes + bytes / 4;
    want = (want + 255) & ~(size_t)255;
    DARBS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    if (buf.ptr) DARBS_CUDA_TRY(ctx, cudaFree(buf.ptr));
    buf.ptr = nullptr;
    buf.bytes = 0;
    DARBS_CUDA_TRY(ctx, cudaMalloc(&buf.ptr, want));
    buf.bytes = want;
    return DARBS_OK;
}

darbs_status reserve_pinned(darbs_cuda_ctx* ctx, size_t bytes) {
    if (bytes <= ctx->pinned_bytes) return DARBS_OK;
    if (ctx->pinned) DARBS_CUDA_TRY(ctx, cudaFreeHost(ctx->pinned));
    ctx->pinned = nullptr;
    ctx->pinned_bytes = 0;
    DARBS_CUDA_TRY(ctx, cudaMallocHost(&ctx->pinned, bytes));
    ctx->pinned_bytes = bytes;
    return DARBS_OK;
}

darbs_status check_launch(darbs_cuda_ctx* ctx, const char* what, int launches) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(ctx, e, what);
    ctx->launches += launches;
    return DARBS_OK;
}

static int pick_fam(const darbs_kernel_spec& s) {
    switch (s.family) {
        case DARBS_GAUSSIAN:
            return s.beta == 2.0 ? FAM_GAUSS2 : FAM_GENERIC;
        case DARBS_HALF_COSINE:
            return s.beta == 2.0 ? FAM_HCOS2 : FAM_GENERIC;
        case DARBS_RAISED_COSINE:
            return (s.beta == 1.0 && s.lobes == 1) ? FAM_RCOS1 : FAM_GENERIC;
        case DARBS_INVERSE_MULTIQUADRATIC:
            return FAM_IMQ;  // eval ignores beta for this family (kernel.cpp:139-145)
        case DARBS_MODULUS_SINC:
            return (s.beta == 1.0 && s.lobes == 1) ? FAM_MSINC1 : FAM_GENERIC;
        default:
            return FAM_GENERIC;
    }
}

static bool is_bounded(int f) {  // kernel.cpp:21-24
    return f == DARBS_HALF_COSINE || f == DARBS_RAISED_COSINE || f == DARBS_MODULUS_SINC;
}

static double u_limit(int family, int lobes) {  // kernel.cpp:27-38
    switch (family) {
        case DARBS_HALF_COSINE:
            return kPiD / 2.0;
        case DARBS_RAISED_COSINE:
            return lobes * kPiD;
        case DARBS_MODULUS_SINC:
            return (lobes + 1) * kPiD / 2.0;
        default:
            return INFINITY;
    }
}

static darbs_status validate_spec(darbs_cuda_ctx* ctx, int family, double beta, double xi, int lobes) {
    // make_kernel kernel.cpp:43-51
    if (family < DARBS_GAUSSIAN || family > DARBS_INVERSE_MULTIQUADRATIC)
        return fail(ctx, DARBS_INVALID_PARAMETER, "unknown kernel family");
    if (!(beta > 0.0) || !std::isfinite(beta))
        return fail(ctx, DARBS_INVALID_PARAMETER, "kernel beta must be positive");
    if (!(xi > 0.0) || !std::isfinite(xi))
        return fail(ctx, DARBS_INVALID_PARAMETER, "kernel xi must be positive");
    if (lobes < 1) return fail(ctx, DARBS_INVALID_PARAMETER, "kernel lobes must be >= 1");
    return DARBS_OK;
}

darbs_status make_kparams(darbs_cuda_ctx* ctx, const darbs_kernel_spec* spec, KParams* out) {
    if (!spec) return fail(ctx, DARBS_INVALID_PARAMETER, "kernel spec is NULL");
    DARBS_TRY(validate_spec(ctx, spec->family, spec->beta, spec->xi, spec->lobes));
    if (!(spec->cutoff > 0.0) || !std::isfinite(spec->cutoff))
        return fail(ctx, DARBS_INVALID_PARAMETER, "kernel cutoff must be positive (use darbs_cuda_make_kernel)");
    KParams kp;
    kp.fam = pick_fam(*spec);
    kp.family = spec->family;
    kp.lobes = spec->lobes;
    kp.unbounded = spec->unbounded ? 1 : 0;
    kp.exact = ctx ? ctx->exact : 1;
    kp.beta = (float)spec->beta;
    kp.xi = (float)spec->xi;
    kp.cutoff = (float)spec->cutoff;
    kp.beta_d = spec->beta;
    kp.xi_d = spec->xi;
    kp.cutoff_d = spec->cutoff;
    kp.scale = (float)family_scale(kp.fam, spec->xi);
    // guard band: 1e-4 in dm2 units, far above the FP32 rounding of the quadratic
    // form (a few ulp of ~10) and of the per-splat threshold.
    kp.band = 1e-4f * kp.scale;
    *out = kp;
    return DARBS_OK;
}

}  // namespace darbs_b200

namespace {

// ---- host <-> device staging -------------------------------------------------
struct Stager {
    darbs_cuda_ctx* ctx;
    darbs_space space;
    int in_slot = 0, out_slot = 0;
    struct Pending {
        void* host;
        const void* dev;
        size_t bytes;
    } pending[8];
    int npending = 0;

    Stager(darbs_cuda_ctx* c, darbs_space s) : ctx(c), space(s) {}

    template <typename T>
    darbs_status in(const T* p, size_t count, const T** out) {
        if (space == DARBS_DEVICE || p == nullptr || count == 0) {
            *out = p;
            return DARBS_OK;
        }
        if (in_slot >= 8) return fail(ctx, DARBS_CUDA_ERROR, "staging slots exhausted");
        DeviceBuffer& b = ctx->stage_in[in_slot++];
        DARBS_TRY(reserve(ctx, b, sizeof(T) * count));
        DARBS_CUDA_TRY(ctx, cudaMemcpyAsync(b.ptr, p, sizeof(T) * count, cudaMemcpyHostToDevice, ctx->stream));
        *out = (const T*)b.ptr;
        return DARBS_OK;
    }
    template <typename T>
    darbs_status out(T* p, size_t count, T** dev) {
        if (space == DARBS_DEVICE || p == nullptr || count == 0) {
            *dev = p;
            return DARBS_OK;
        }
        if (out_slot >= 8) return fail(ctx, DARBS_CUDA_ERROR, "staging slots exhausted");
        DeviceBuffer& b = ctx->stage_out[out_slot++];
        DARBS_TRY(reserve(ctx, b, sizeof(T) * count));
        *dev = (T*)b.ptr;
        pending[npending++] = {p, b.ptr, sizeof(T) * count};
        return DARBS_OK;
    }
    // Upload that the call consumes late: runs on the context's copy stream, behind everything
    // already queued on the main stream (the previous call may still read the staging buffer);
    // the caller puts await_late() in front of the first kernel that reads it.
    template <typename T>
    darbs_status in_late(const T* p, size_t count, const T** out) {
        if (space == DARBS_DEVICE || p == nullptr || count == 0) {
            *out = p;
            return DARBS_OK;
        }
        if (in_slot >= 8) return fail(ctx, DARBS_CUDA_ERROR, "staging slots exhausted");
        DeviceBuffer& b = ctx->stage_in[in_slot++];
        DARBS_TRY(reserve(ctx, b, sizeof(T) * count));
        DARBS_CUDA_TRY(ctx, cudaEventRecord(ctx->copy_begin, ctx->stream));
        DARBS_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->copy_stream, ctx->copy_begin, 0));
        DARBS_CUDA_TRY(ctx, cudaMemcpyAsync(b.ptr, p, sizeof(T) * count, cudaMemcpyHostToDevice, ctx->copy_stream));
        DARBS_CUDA_TRY(ctx, cudaEventRecord(ctx->copy_done, ctx->copy_stream));
        late = true;
        *out = (const T*)b.ptr;
        return DARBS_OK;
    }
    darbs_status await_late() {
        if (late) DARBS_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, ctx->copy_done, 0));
        late = false;
        return DARBS_OK;
    }
    bool late = false;
    // in-out host array (accumulators)
    template <typename T>
    darbs_status inout(T* p, size_t count, T** dev) {
        DARBS_TRY(out(p, count, dev));
        if (space == DARBS_HOST && p && count)
            DARBS_CUDA_TRY(ctx, cudaMemcpyAsync(*dev, p, sizeof(T) * count, cudaMemcpyHostToDevice, ctx->stream));
        return DARBS_OK;
    }
    darbs_status finish() {
        if (space == DARBS_DEVICE || npending == 0) return DARBS_OK;
        for (int i = 0; i < npending; ++i)
            DARBS_CUDA_TRY(ctx, cudaMemcpyAsync(pending[i].host, pending[i].dev, pending[i].bytes,
                                                cudaMemcpyDeviceToHost, ctx->stream));
        DARBS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
        return DARBS_OK;
    }
};

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
        else prev = -1;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// ---- stage timing ------------------------------------------------------------
enum { ST_PREPROCESS = 0, ST_BINNING, ST_RENDER_FWD, ST_LOSS, ST_RENDER_BWD, ST_PREPROCESS_BWD, ST_ADAM, ST_CULL };

struct StageScope {
    darbs_cuda_ctx* ctx;
    int stage;
    StageScope(darbs_cuda_ctx* c, int s) : ctx(c), stage(s) {
        if (ctx->timing) cudaEventRecord(ctx->timer.ev[2 * stage], ctx->stream);
    }
    ~StageScope() {
        if (ctx->timing) cudaEventRecord(ctx->timer.ev[2 * stage + 1], ctx->stream);
    }
};

void reset_stage_marks(darbs_cuda_ctx* ctx, std::initializer_list<int> stages) {
    if (!ctx->timing) return;
    for (int s = 0; s < 8; ++s) ctx->stage_ms[s] = -1.0;  // -1: not part of the last call
    for (int s : stages) ctx->stage_ms[s] = -2.0;         // -2: events pending
}

#define CTX_OR_FAIL(ctx) \
    if (!(ctx)) return fail(nullptr, DARBS_INVALID_PARAMETER, "context is NULL")

// ---- forward on device arrays ------------------------------------------------
darbs_status forward_device(darbs_cuda_ctx* ctx, const KParams& kp, int64_t n, const float* mu2,
                            const float* conic, const float* radius, const float* depth,
                            const float* opacity, const float* rgb, const int32_t* valid, int width,
                            int height, const float bg[3], float* image, int32_t* contributors,
                            bool preprocessed = false) {
    // preprocessed: the fused preprocess of evaluate_view already left the tile rectangles, depth
    // keys and packed records (binning_begin's sinks), so rect_kernel and pack_kernel are skipped
    const size_t px = (size_t)width * height;
    {
        StageScope ts(ctx, ST_BINNING);
        ctx->tile_order_wanted = ctx->tile_order_lpt != 0;  // a forward follows: its CTAs take the long tiles first
        const darbs_status st_bin = run_binning(ctx, n, mu2, conic, radius, depth, valid, width, height, preprocessed);
        ctx->tile_order_wanted = false;
        DARBS_TRY(st_bin);
    }
    {
        StageScope ts(ctx, ST_CULL);
        if (!preprocessed) DARBS_TRY(launch_pack(ctx, kp, n, mu2, conic, opacity, rgb));
        DARBS_TRY(launch_cull(ctx, kp));
    }
    // prefetched uploads may start here: from now on the stream holds a few long kernels, whose
    // launches a bulk PCIe transfer cannot delay (it does delay the many short ones of the sort)
    cudaEventRecord(ctx->after_cull, ctx->stream);
    ctx->have_after_cull = true;
    DARBS_TRY(reserve(ctx, ctx->t_final, sizeof(float) * (px ? px : 1)));
    DARBS_TRY(reserve(ctx, ctx->processed, sizeof(int32_t) * (px ? px : 1)));
    if (!image) {
        DARBS_TRY(reserve(ctx, ctx->image, sizeof(float) * 3 * (px ? px : 1)));
        image = (float*)ctx->image.ptr;
    }
    if (!contributors) {
        DARBS_TRY(reserve(ctx, ctx->contributors, sizeof(int32_t) * (px ? px : 1)));
        contributors = (int32_t*)ctx->contributors.ptr;
    }
    {
        StageScope ts(ctx, ST_RENDER_FWD);
        DARBS_TRY(launch_render_fwd(ctx, kp, width, height, bg, image, (float*)ctx->t_final.ptr,
                                    (int32_t*)ctx->processed.ptr, contributors));
    }
    ctx->have_forward = true;
    ctx->fwd_family = kp.family;
    ctx->fwd_lobes = kp.lobes;
    ctx->fwd_beta = kp.beta_d;
    ctx->fwd_xi = kp.xi_d;
    ctx->fwd_contrib = contributors;
    ctx->fwd_n = n;
    ctx->fwd_w = width;
    ctx->fwd_h = height;
    memcpy(ctx->fwd_bg, bg, sizeof(float) * 3);
    return DARBS_OK;
}

}  // namespace

// =============================================================================
extern "C" {

const char* darbs_cuda_version(void) { return "darbs-b200 0.1 (sm_100a)"; }

darbs_status darbs_cuda_create(int device, darbs_cuda_ctx** out_ctx) {
    if (!out_ctx) return fail(nullptr, DARBS_INVALID_PARAMETER, "out_ctx is NULL");
    *out_ctx = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        return fail(nullptr, DARBS_CUDA_ERROR,
                    std::string("no usable CUDA device (there is no CPU fallback): ") +
                        (e != cudaSuccess ? cudaGetErrorString(e) : "device count is 0"));
    if (device < 0 || device >= count) return fail(nullptr, DARBS_INVALID_PARAMETER, "device index out of range");
    cudaDeviceProp prop;
    e = cudaGetDeviceProperties(&prop, device);
    if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaGetDeviceProperties");
    if (prop.major != 10)
        return fail(nullptr, DARBS_CUDA_ERROR,
                    "this library is built for sm_100a (B200) only; device is sm_" +
                        std::to_string(prop.major) + std::to_string(prop.minor));
    darbs_cuda_ctx* ctx = new (std::nothrow) darbs_cuda_ctx();
    if (!ctx) return fail(nullptr, DARBS_CUDA_ERROR, "out of host memory");
    ctx->device = device;
    ctx->sm_count = prop.multiProcessorCount;
    if (const char* e = getenv("DARBS_TILE_ORDER")) ctx->tile_order_lpt = atoi(e);
    DeviceGuard guard(device);
    e = cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete ctx;
        return cuda_fail(nullptr, e, "cudaStreamCreate");
    }
    ctx->stream = ctx->own_stream;
    cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&ctx->aux_stream, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&ctx->ranges_ready, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->order_ready, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->copy_begin, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->copy_done, cudaEventDisableTiming);
    for (int i = 0; i < 16; ++i) cudaEventCreate(&ctx->timer.ev[i]);
    ctx->timer.created = true;
    cudaEventCreateWithFlags(&ctx->after_cull, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->k_ready, cudaEventDisableTiming);
    for (int i = 0; i < 2; ++i) {
        cudaEventCreateWithFlags(&ctx->target_done[i], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&ctx->target_read[i], cudaEventDisableTiming);
    }
    for (int i = 0; i < kLossRing; ++i) {
        cudaMallocHost(&ctx->loss_ring[i].host, 64);
        cudaEventCreateWithFlags(&ctx->loss_ring[i].done, cudaEventDisableTiming);
    }
    darbs_status st = reserve(ctx, ctx->counters, 1024);  // 32 scalar slots + kSlotsK partial sums of K
    if (st == DARBS_OK) st = reserve_pinned(ctx, 256);
    if (st == DARBS_OK && cudaMemsetAsync(ctx->counters.ptr, 0, 1024, ctx->stream) != cudaSuccess)
        st = DARBS_CUDA_ERROR;
    if (st != DARBS_OK) {
        g_create_error = ctx->last_error;
        darbs_cuda_destroy(ctx);
        return st;
    }
    *out_ctx = ctx;
    return DARBS_OK;
}

void darbs_cuda_destroy(darbs_cuda_ctx* ctx) {
    if (!ctx) return;
    DeviceGuard guard(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    destroy_comm(ctx);
    DeviceBuffer* bufs[] = {&ctx->recs, &ctx->rects, &ctx->depth_keys, &ctx->order,
                            &ctx->tile_keys, &ctx->tile_vals, &ctx->ranges, &ctx->streams, &ctx->stream_count, &ctx->sort_ws, &ctx->tile_status, &ctx->tile_order,
                            &ctx->counters, &ctx->t_final, &ctx->processed, &ctx->contributors,
                            &ctx->image, &ctx->valid, &ctx->splat_grads, &ctx->splat_grads_fx, &ctx->grad_image, &ctx->loss_maps};
    for (DeviceBuffer* b : bufs)
        if (b->ptr) cudaFree(b->ptr);
    for (int i = 0; i < 8; ++i) {
        if (ctx->stage_in[i].ptr) cudaFree(ctx->stage_in[i].ptr);
        if (ctx->stage_out[i].ptr) cudaFree(ctx->stage_out[i].ptr);
    }
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    if (ctx->timer.created)
        for (int i = 0; i < 16; ++i) cudaEventDestroy(ctx->timer.ev[i]);
    for (int i = 0; i < kLossRing; ++i) {
        if (ctx->loss_ring[i].host) cudaFreeHost(ctx->loss_ring[i].host);
        if (ctx->loss_ring[i].done) cudaEventDestroy(ctx->loss_ring[i].done);
    }
    if (ctx->after_cull) cudaEventDestroy(ctx->after_cull);
    if (ctx->k_ready) cudaEventDestroy(ctx->k_ready);
    for (int i = 0; i < 2; ++i) {
        if (ctx->target_done[i]) cudaEventDestroy(ctx->target_done[i]);
        if (ctx->target_read[i]) cudaEventDestroy(ctx->target_read[i]);
        if (ctx->target_stage[i].ptr) cudaFree(ctx->target_stage[i].ptr);
    }
    if (ctx->copy_begin) cudaEventDestroy(ctx->copy_begin);
    if (ctx->copy_done) cudaEventDestroy(ctx->copy_done);
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    if (ctx->aux_stream) cudaStreamDestroy(ctx->aux_stream);
    if (ctx->ranges_ready) cudaEventDestroy(ctx->ranges_ready);
    if (ctx->order_ready) cudaEventDestroy(ctx->order_ready);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;
}

const char* darbs_cuda_last_error(const darbs_cuda_ctx* ctx) {
    return ctx ? ctx->last_error.c_str() : g_create_error.c_str();
}

darbs_status darbs_cuda_set_stream(darbs_cuda_ctx* ctx, void* cuda_stream) {
    CTX_OR_FAIL(ctx);
    DeviceGuard guard(ctx->device);
    cudaStream_t next = cuda_stream ? (cudaStream_t)cuda_stream : ctx->own_stream;
    // binding the stream the context already runs on is free (callers re-bind before every call
    // when they share the stream with other libraries; it may also be capturing a graph)
    if (next == ctx->stream) return DARBS_OK;
    DARBS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    ctx->stream = next;
    return DARBS_OK;
}

darbs_status darbs_cuda_synchronize(darbs_cuda_ctx* ctx) {
    CTX_OR_FAIL(ctx);
    DeviceGuard guard(ctx->device);
    DARBS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return DARBS_OK;
}

int64_t darbs_cuda_launch_count(const darbs_cuda_ctx* ctx) { return ctx ? ctx->launches : 0; }

darbs_status darbs_cuda_set_exact_decisions(darbs_cuda_ctx* ctx, int enabled) {
    CTX_OR_FAIL(ctx);
    ctx->exact = enabled ? 1 : 0;
    return DARBS_OK;
}

// ---- device memory ---------------------------------------------------------------

darbs_status darbs_cuda_device_alloc(darbs_cuda_ctx* ctx, uint64_t bytes, void** out_ptr) {
    CTX_OR_FAIL(ctx);
    if (!out_ptr) return fail(ctx, DARBS_INVALID_PARAMETER, "device_alloc: out_ptr is NULL");
    *out_ptr = nullptr;
    DeviceGuard guard(ctx->device);
    DARBS_CUDA_TRY(ctx, cudaMalloc(out_ptr, bytes ? (size_t)bytes : 1));
    return DARBS_OK;
}

darbs_status darbs_cuda_device_free(darbs_cuda_ctx* ctx, void* ptr) {
    CTX_OR_FAIL(ctx);
    if (!ptr) return DARBS_OK;
    DeviceGuard guard(ctx->device);
    DARBS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    DARBS_CUDA_TRY(ctx, cudaFree(ptr));
    return DARBS_OK;
}

darbs_status darbs_cuda_upload(darbs_cuda_ctx* ctx, void* dst_device, const void* src_host, uint64_t bytes) {
    CTX_OR_FAIL(ctx);
    if (bytes == 0) return DARBS_OK;
    if (!dst_device || !src_host) return fail(ctx, DARBS_INVALID_PARAMETER, "upload: NULL pointer");
    DeviceGuard guard(ctx->device);
    // pageable source memory is staged by the runtime before the call returns
    DARBS_CUDA_TRY(ctx, cudaMemcpyAsync(dst_device, src_host, (size_t)bytes, cudaMemcpyHostToDevice, ctx->stream));
    DARBS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return DARBS_OK;
}

darbs_status darbs_cuda_download(darbs_cuda_ctx* ctx, void* dst_host, const void* src_device, uint64_t bytes) {
    CTX_OR_FAIL(ctx);
    if (bytes == 0) return DARBS_OK;
    if (!dst_host || !src_device) return fail(ctx, DARBS_INVALID_PARAMETER, "download: NULL pointer");
    DeviceGuard guard(ctx->device);
    DARBS_CUDA_TRY(ctx, cudaMemcpyAsync(dst_host, src_device, (size_t)bytes, cudaMemcpyDeviceToHost, ctx->stream));
    DARBS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return DARBS_OK;
}

darbs_status darbs_cuda_device_zero(darbs_cuda_ctx* ctx, void* ptr, uint64_t bytes) {
    CTX_OR_FAIL(ctx);
    if (bytes == 0) return DARBS_OK;
    if (!ptr) return fail(ctx, DARBS_INVALID_PARAMETER, "device_zero: NULL pointer");
    DeviceGuard guard(ctx->device);
    DARBS_CUDA_TRY(ctx, cudaMemsetAsync(ptr, 0, (size_t)bytes, ctx->stream));
    return DARBS_OK;
}

// ---- kernel family ------------------------------------------------------------

darbs_status darbs_cuda_make_kernel(int family, double beta, double xi, int lobes, darbs_kernel_spec* out) {
    if (!out) return fail(nullptr, DARBS_INVALID_PARAMETER, "out is NULL");
    DARBS_TRY(validate_spec(nullptr, family, beta, xi, lobes));
    out->family = family;
    out->beta = beta;
    out->xi = xi;
    out->lobes = lobes;
    out->unbounded = is_bounded(family) ? 0 : 1;
    if (out->unbounded)
        out->cutoff = 3.0 * 3.0;  // kRenderCutoffDm kernel.cpp:19, :58-59
    else
        out->cutoff = std::pow(xi * u_limit(family, lobes), 2.0 / beta);  // kernel.cpp:61-62
    return DARBS_OK;
}

darbs_status darbs_cuda_kernel_preset(const char* name, darbs_kernel_spec* out) {
    if (!name || !out) return fail(nullptr, DARBS_INVALID_PARAMETER, "NULL argument");
    // kernel.cpp:223-240
    if (!strcmp(name, "gaussian")) return darbs_cuda_make_kernel(DARBS_GAUSSIAN, 2.0, 2.0, 1, out);
    if (!strcmp(name, "half-cosine-sq")) return darbs_cuda_make_kernel(DARBS_HALF_COSINE, 2.0, 18.0 / kPiD, 1, out);
    if (!strcmp(name, "raised-cosine")) return darbs_cuda_make_kernel(DARBS_RAISED_COSINE, 1.0, 2.5 / kPiD, 1, out);
    if (!strcmp(name, "mod-sinc")) return darbs_cuda_make_kernel(DARBS_MODULUS_SINC, 1.0, 3.0 / kPiD, 1, out);
    if (!strcmp(name, "inv-multiquadratic"))
        return darbs_cuda_make_kernel(DARBS_INVERSE_MULTIQUADRATIC, 2.0, 1.0, 1, out);
    return fail(nullptr, DARBS_INVALID_PARAMETER, std::string("unknown kernel preset: ") + name);
}

double darbs_cuda_default_psi(const char* name) {
    // kPsiDefaults psi_table.hpp:20-26
    if (!name) return -1.0;
    if (!strcmp(name, "gaussian")) return 1.0;
    if (!strcmp(name, "half-cosine-sq")) return 1.36;
    if (!strcmp(name, "raised-cosine")) return 0.6552;
    if (!strcmp(name, "mod-sinc")) return 1.1762;
    if (!strcmp(name, "inv-multiquadratic")) return 1.6054;
    return -1.0;
}

darbs_status darbs_cuda_eval(darbs_cuda_ctx* ctx, const darbs_kernel_spec* kernel, int64_t n,
                             const float* dm2, float* weight, float* dweight_ddm2, int exact,
                             darbs_space space) {
    CTX_OR_FAIL(ctx);
    DeviceGuard guard(ctx->device);
    KParams kp;
    DARBS_TRY(make_kparams(ctx, kernel, &kp));
    if (space == DARBS_HOST) {
        for (int64_t i = 0; i < n; ++i)
            if (dm2[i] < 0.f || !std::isfinite(dm2[i]))  // kernel.cpp:128-130
                return fail(ctx, DARBS_INVALID_PARAMETER, "eval: dm2 must be finite and non-negative");
    }
    Stager st(ctx, space);
    const float* d_in;
    float *d_w, *d_dw;
    DARBS_TRY(st.in(dm2, (size_t)n, &d_in));
    DARBS_TRY(st.out(weight, (size_t)n, &d_w));
    DARBS_TRY(st.out(dweight_ddm2, (size_t)n, &d_dw));
    DARBS_TRY(launch_eval(ctx, kp, n, d_in, d_w, d_dw, exact));
    return st.finish();
}

// ---- rasterizer -----------------------------------------------------------------

darbs_status darbs_cuda_bin(darbs_cuda_ctx* ctx, int64_t n, const float* mu2, const float* conic,
                            const float* radius, const float* depth, int width, int height,
                            int64_t* num_entries, int32_t* tile_ranges, int32_t* point_list,
                            uint64_t* sort_keys, int32_t* depth_order, int64_t capacity,
                            darbs_space space) {
    CTX_OR_FAIL(ctx);
    if (n < 0 || width < 0 || height < 0) return fail(ctx, DARBS_INVALID_PARAMETER, "negative size");
    DeviceGuard guard(ctx->device);
    Stager st(ctx, space);
    const float *d_mu2, *d_conic, *d_radius, *d_depth;
    DARBS_TRY(st.in(mu2, 2 * (size_t)n, &d_mu2));
    DARBS_TRY(st.in(conic, 3 * (size_t)n, &d_conic));
    DARBS_TRY(st.in(radius, (size_t)n, &d_radius));
    DARBS_TRY(st.in(depth, (size_t)n, &d_depth));
    ctx->have_forward = false;
    DARBS_TRY(run_binning(ctx, n, d_mu2, d_conic, d_radius, d_depth, nullptr, width, height));
    const int64_t k = ctx->fwd_entries;
    if (num_entries) *num_entries = k;
    const bool fits = k <= capacity;
    const size_t tiles = (size_t)ctx->tiles_x * ctx->tiles_y;
    int32_t *d_ranges, *d_plist, *d_order;
    uint64_t* d_keys;
    DARBS_TRY(st.out(tile_ranges, 2 * tiles, &d_ranges));
    DARBS_TRY(st.out(fits ? point_list : nullptr, (size_t)k, &d_plist));
    DARBS_TRY(st.out(fits ? sort_keys : nullptr, (size_t)k, &d_keys));
    DARBS_TRY(st.out(depth_order, (size_t)n, &d_order));
    DARBS_TRY(export_bins(ctx, n, d_ranges, d_plist, d_keys, d_order));
    return st.finish();
}

darbs_status darbs_cuda_forward(darbs_cuda_ctx* ctx, const darbs_kernel_spec* kernel, int64_t n,
                                const float* mu2, const float* conic, const float* radius,
                                const float* depth, const float* opacity, const float* rgb, int width,
                                int height, const float background[3], float* image, float* t_final,
                                int32_t* processed, int32_t* contributors, int32_t* skipped_nonfinite,
                                darbs_space space) {
    CTX_OR_FAIL(ctx);
    if (n < 0 || width < 0 || height < 0) return fail(ctx, DARBS_INVALID_PARAMETER, "negative size");
    if (!background) return fail(ctx, DARBS_INVALID_PARAMETER, "background is NULL");
    if (n > 0 && (!mu2 || !conic || !radius || !depth || !opacity || !rgb))
        return fail(ctx, DARBS_INVALID_PARAMETER, "splat array is NULL");
    DeviceGuard guard(ctx->device);
    KParams kp;
    DARBS_TRY(make_kparams(ctx, kernel, &kp));
    reset_stage_marks(ctx, {ST_BINNING, ST_CULL, ST_RENDER_FWD});
    Stager st(ctx, space);
    const float *d_mu2, *d_conic, *d_radius, *d_depth, *d_opacity, *d_rgb;
    DARBS_TRY(st.in(mu2, 2 * (size_t)n, &d_mu2));
    DARBS_TRY(st.in(conic, 3 * (size_t)n, &d_conic));
    DARBS_TRY(st.in(radius, (size_t)n, &d_radius));
    DARBS_TRY(st.in(depth, (size_t)n, &d_depth));
    DARBS_TRY(st.in(opacity, (size_t)n, &d_opacity));
    DARBS_TRY(st.in(rgb, 3 * (size_t)n, &d_rgb));
    const size_t px = (size_t)width * height;
    float* d_image;
    int32_t* d_contrib;
    DARBS_TRY(st.out(image, 3 * px, &d_image));
    DARBS_TRY(st.out(contributors, px, &d_contrib));
    ctx->have_forward = false;
    DARBS_TRY(forward_device(ctx, kp, n, d_mu2, d_conic, d_radius, d_depth, d_opacity, d_rgb, nullptr,
                             width, height, background, d_image, d_contrib));
    // t_final / processed stay resident for backward; copy out on request
    if (space == DARBS_DEVICE) {
        if (t_final && px)
            DARBS_CUDA_TRY(ctx, cudaMemcpyAsync(t_final, ctx->t_final.ptr, sizeof(float) * px,
                                                cudaMemcpyDeviceToDevice, ctx->stream));
        if (processed && px)
            DARBS_CUDA_TRY(ctx, cudaMemcpyAsync(processed, ctx->processed.ptr, sizeof(int32_t) * px,
                                                cudaMemcpyDeviceToDevice, ctx->stream));
    } else {
        if (t_final && px)
            DARBS_CUDA_TRY(ctx, cudaMemcpyAsync(t_final, ctx->t_final.ptr, sizeof(float) * px,
                                                cudaMemcpyDeviceToHost, ctx->stream));
        if (processed && px)
            DARBS_CUDA_TRY(ctx, cudaMemcpyAsync(processed, ctx->processed.ptr, sizeof(int32_t) * px,
                                                cudaMemcpyDeviceToHost, ctx->stream));
    }
    if (skipped_nonfinite) {
        const unsigned long long* sc = (const unsigned long long*)ctx->counters.ptr + 8;
        DARBS_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->pinned, sc, sizeof(unsigned long long) * 2,
                                            cudaMemcpyDeviceToHost, ctx->stream));
        DARBS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
        *skipped_nonfinite = (int32_t)((unsigned long long*)ctx->pinned)[1];
    }
    return st.finish();
}

darbs_status darbs_cuda_backward(darbs_cuda_ctx* ctx, const darbs_kernel_spec* kernel, int grad_width,
                                 int grad_height, const float* grad_image, int64_t n, const float* mu2,
                                 const float* conic, const float* opacity, const float* rgb,
                                 float* grads, darbs_space space) {
    CTX_OR_FAIL(ctx);
    // rasterizer.cpp:151-154
    if (!ctx->have_forward || grad_width != ctx->fwd_w || grad_height != ctx->fwd_h || n != ctx->fwd_n)
        return fail(ctx, DARBS_CONTRACT_VIOLATION, "backward: aux does not match this forward call");
    if (!grad_image && (size_t)grad_width * grad_height > 0)
        return fail(ctx, DARBS_INVALID_PARAMETER, "grad_image is NULL");
    if (!grads && n > 0) return fail(ctx, DARBS_INVALID_PARAMETER, "grads is NULL");
    DeviceGuard guard(ctx->device);
    KParams kp;
    DARBS_TRY(make_kparams(ctx, kernel, &kp));
    if (kp.family != ctx->fwd_family || kp.lobes != ctx->fwd_lobes || kp.beta_d != ctx->fwd_beta ||
        kp.xi_d != ctx->fwd_xi)
        return fail(ctx, DARBS_CONTRACT_VIOLATION, "backward: not the kernel the forward call ran with");
    reset_stage_marks(ctx, {ST_RENDER_BWD});
    Stager st(ctx, space);
    const size_t px = (size_t)grad_width * grad_height;
    const float* d_gimg;
    DARBS_TRY(st.in(grad_image, 3 * px, &d_gimg));
    (void)mu2, (void)conic, (void)opacity, (void)rgb;  // not read: see the header
    float* d_grads;
    DARBS_TRY(st.out(grads, (size_t)DARBS_GRADS_PER_SPLAT * (size_t)n, &d_grads));
    {
        StageScope ts(ctx, ST_RENDER_BWD);
        DARBS_TRY(launch_render_bwd(ctx, kp, grad_width, grad_height, ctx->fwd_bg, d_gimg,
                                    (const float*)ctx->t_final.ptr, (const int32_t*)ctx->processed.ptr, n));
    }
    DARBS_TRY(launch_export_grads(ctx, n, d_grads));
    return st.finish();
}

// ---- geometry -------------------------------------------------------------------

darbs_status darbs_cuda_realize(darbs_cuda_ctx* ctx, int64_t n, const float* raw, float* prims,
                                darbs_space space) {
    CTX_OR_FAIL(ctx);
    DeviceGuard guard(ctx->device);
    Stager st(ctx, space);
    const float* d_raw;
    float* d_prims;
    DARBS_TRY(st.in(raw, 14 * (size_t)n, &d_raw));
    DARBS_TRY(st.out(prims, 14 * (size_t)n, &d_prims));
    DARBS_TRY(launch_realize(ctx, n, d_raw, d_prims));
    return st.finish();
}

// the three loss sums as the device left them: doubles, or int64 fixed point in the deterministic mode
static void read_loss_sums(const void* src, bool fixed_point, double out[3]) {
    for (int i = 0; i < 3; ++i) {
        if (fixed_point) {
            long long v;
            std::memcpy(&v, (const char*)src + 8 * i, 8);
            out[i] = (double)v / kFixedScale;
        } else {
            std::memcpy(&out[i], (const char*)src + 8 * i, 8);
        }
    }
}

static darbs_status read_flags(darbs_cuda_ctx* ctx, const int* d_flags, int out[2]) {
    DARBS_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->pinned, d_flags, sizeof(int) * 2, cudaMemcpyDeviceToHost,
                                        ctx->stream));
    DARBS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    out[0] = ((int*)ctx->pinned)[0];
    out[1] = ((int*)ctx->pinned)[1];
    return DARBS_OK;
}

darbs_status darbs_cuda_project(darbs_cuda_ctx* ctx, const darbs_kernel_spec* kernel, double psi,
                                double dilation, int64_t n, const float* prims, const double* camera,
                                int32_t* valid, float* mu2, float* cov2, float* conic, float* radius,
                                float* depth, darbs_space space) {
    CTX_OR_FAIL(ctx);
    if (!camera) return fail(ctx, DARBS_INVALID_PARAMETER, "camera is NULL");
    if (n > 0 && (!prims || !mu2 || !conic || !radius || !depth))
        return fail(ctx, DARBS_INVALID_PARAMETER, "NULL array");
    DeviceGuard guard(ctx->device);
    KParams kp;
    DARBS_TRY(make_kparams(ctx, kernel, &kp));
    Stager st(ctx, space);
    const float* d_prims;
    int32_t* d_valid;
    float *d_mu2, *d_cov2, *d_conic, *d_radius, *d_depth;
    DARBS_TRY(st.in(prims, 14 * (size_t)n, &d_prims));
    DARBS_TRY(st.out(valid, (size_t)n, &d_valid));
    DARBS_TRY(st.out(mu2, 2 * (size_t)n, &d_mu2));
    DARBS_TRY(st.out(cov2, 3 * (size_t)n, &d_cov2));
    DARBS_TRY(st.out(conic, 3 * (size_t)n, &d_conic));
    DARBS_TRY(st.out(radius, (size_t)n, &d_radius));
    DARBS_TRY(st.out(depth, (size_t)n, &d_depth));
    int* d_flags = (int*)((unsigned long long*)ctx->counters.ptr + 12);
    DARBS_CUDA_TRY(ctx, cudaMemsetAsync(d_flags, 0, sizeof(int) * 2, ctx->stream));
    DARBS_TRY(launch_project(ctx, kp, psi, dilation, n, d_prims, false, make_camera(camera), d_valid,
                             d_mu2, d_cov2, d_conic, d_radius, d_depth, nullptr, nullptr, d_flags));
    DARBS_TRY(st.finish());
    int flags[2];
    DARBS_TRY(read_flags(ctx, d_flags, flags));
    // the order the reference would throw in for one primitive: scale (geometry.cpp:10),
    // psi (:44), degenerate covariance (:53)
    if (flags[0] & 1) return fail(ctx, DARBS_INVALID_PARAMETER, "covariance_from_scale_rot: scale must be positive");
    if (!(psi > 0.0) && n > 0 && flags[1] > 0) return fail(ctx, DARBS_INVALID_PARAMETER, "apply_psi: psi must be positive");
    if (flags[0] & 2) return fail(ctx, DARBS_NUMERIC_ERROR, "conic_and_radius: covariance not positive definite");
    return DARBS_OK;
}

darbs_status darbs_cuda_backward_projection(darbs_cuda_ctx* ctx, double psi, int64_t n,
                                            const float* grad_cov2, const float* grad_mu2,
                                            const float* prims, const double* camera, float* d_mu,
                                            float* d_scale, float* d_rot, darbs_space space) {
    CTX_OR_FAIL(ctx);
    if (!camera) return fail(ctx, DARBS_INVALID_PARAMETER, "camera is NULL");
    DeviceGuard guard(ctx->device);
    Stager st(ctx, space);
    const float *d_gc, *d_gm, *d_prims;
    float *o_mu, *o_scale, *o_rot;
    DARBS_TRY(st.in(grad_cov2, 4 * (size_t)n, &d_gc));
    DARBS_TRY(st.in(grad_mu2, 2 * (size_t)n, &d_gm));
    DARBS_TRY(st.in(prims, 14 * (size_t)n, &d_prims));
    DARBS_TRY(st.out(d_mu, 3 * (size_t)n, &o_mu));
    DARBS_TRY(st.out(d_scale, 3 * (size_t)n, &o_scale));
    DARBS_TRY(st.out(d_rot, 4 * (size_t)n, &o_rot));
    DARBS_TRY(launch_backward_projection(ctx, psi, n, d_gc, d_gm, d_prims, make_camera(camera), o_mu,
                                         o_scale, o_rot));
    return st.finish();
}

// ---- training step ----------------------------------------------------------------

darbs_status darbs_cuda_evaluate_view(darbs_cuda_ctx* ctx, const darbs_kernel_spec* kernel, double psi,
                                      int64_t n, const float* raw_params, const double* camera,
                                      const float background[3], const float* target, double lambda,
                                      const float* grad_image, float* param_grads, float* image_out,
                                      double loss_out[4], darbs_space param_space,
                                      darbs_space image_space) {
    CTX_OR_FAIL(ctx);
    if (!camera || !background) return fail(ctx, DARBS_INVALID_PARAMETER, "camera/background is NULL");
    if ((target != nullptr) == (grad_image != nullptr))
        return fail(ctx, DARBS_INVALID_PARAMETER, "pass exactly one of target / grad_image");
    if (target && !(lambda >= 0.0 && lambda <= 1.0))
        return fail(ctx, DARBS_INVALID_PARAMETER, "lambda must lie in [0, 1]");
    if (n <= 0 || !raw_params) return fail(ctx, DARBS_INVALID_PARAMETER, "empty primitive set");
    if (!(psi > 0.0)) return fail(ctx, DARBS_INVALID_PARAMETER, "apply_psi: psi must be positive");
    DeviceGuard guard(ctx->device);
    KParams kp;
    DARBS_TRY(make_kparams(ctx, kernel, &kp));
    const CameraD cam = make_camera(camera);
    const int width = cam.width, height = cam.height;
    if (width <= 0 || height <= 0) return fail(ctx, DARBS_INVALID_PARAMETER, "camera has no pixels");
    const size_t px = (size_t)width * height, nn = (size_t)n;
    reset_stage_marks(ctx, {ST_PREPROCESS, ST_BINNING, ST_CULL, ST_RENDER_FWD, ST_LOSS, ST_RENDER_BWD, ST_PREPROCESS_BWD});

    Stager st(ctx, param_space);
    Stager sti(ctx, image_space);
    sti.in_slot = 4;   // the two stagers share the context's staging slots
    sti.out_slot = 4;
    const float *d_raw, *d_target, *d_gimg;
    float *d_pgrads, *d_image;
    DARBS_TRY(st.in(raw_params, 14 * nn, &d_raw));
    int staged = -1;
    if (target && image_space == DARBS_HOST)
        for (int i = 0; i < 2; ++i)
            if (ctx->target_src[i] == target && ctx->target_stage[i].bytes >= sizeof(float) * 3 * px) staged = i;
    if (staged >= 0) {
        d_target = (const float*)ctx->target_stage[staged].ptr;  // uploaded by darbs_cuda_prefetch_target
        ctx->target_src[staged] = nullptr;
    } else {
        DARBS_TRY(sti.in_late(target, 3 * px, &d_target));  // not needed before the loss: overlaps the forward
    }
    DARBS_TRY(sti.in(grad_image, 3 * px, &d_gimg));
    const bool overwrite = !ctx->accumulate;
    ctx->accumulate = 1;
    if (overwrite)
        DARBS_TRY(st.out(param_grads, 14 * nn, &d_pgrads));
    else
        DARBS_TRY(st.inout(param_grads, 14 * nn, &d_pgrads));
    DARBS_TRY(sti.out(image_out, 3 * px, &d_image));

    // internal SoA of the projected splats (one slot each; no compaction)
    DARBS_TRY(reserve(ctx, ctx->valid, sizeof(int32_t) * nn + sizeof(float) * 11 * nn));
    int32_t* d_valid = (int32_t*)ctx->valid.ptr;
    float* d_mu2 = (float*)(d_valid + nn);
    float* d_conic = d_mu2 + 2 * nn;
    float* d_radius = d_conic + 3 * nn;
    float* d_depth = d_radius + nn;
    float* d_opacity = d_depth + nn;
    float* d_rgb = d_opacity + nn;
    int* d_flags = (int*)((unsigned long long*)ctx->counters.ptr + 12);
    double* d_sums = (double*)((unsigned long long*)ctx->counters.ptr + 14);
    ctx->have_forward = false;
    {
        StageScope ts(ctx, ST_PREPROCESS);
        DARBS_CUDA_TRY(ctx, cudaMemsetAsync(d_flags, 0, sizeof(int) * 2, ctx->stream));
        SplatSinks sinks;
        DARBS_TRY(binning_begin(ctx, n, width, height, &sinks));
        DARBS_TRY(reserve(ctx, ctx->recs, sizeof(float4) * kRecVecs * nn));
        sinks.recs = (float4*)ctx->recs.ptr;
        DARBS_TRY(launch_project(ctx, kp, psi, DARBS_DILATION, n, d_raw, true, cam, d_valid, d_mu2,
                                 nullptr, d_conic, d_radius, d_depth, d_opacity, d_rgb, d_flags, &sinks));
    }
    if (!d_image) {
        DARBS_TRY(reserve(ctx, ctx->image, sizeof(float) * 3 * px));
        d_image = (float*)ctx->image.ptr;
    }
    DARBS_TRY(forward_device(ctx, kp, n, d_mu2, d_conic, d_radius, d_depth, d_opacity, d_rgb, d_valid,
                             width, height, background, d_image, nullptr, /*preprocessed=*/true));
    DARBS_TRY(sti.await_late());
    if (staged >= 0) DARBS_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, ctx->target_done[staged], 0));
    if (target) {
        StageScope ts(ctx, ST_LOSS);
        // without param_grads nothing consumes dL/dimage: values only (fit_scene's evaluate(false), fit3d.cpp:131)
        float* d_lgrad = nullptr;
        if (param_grads) {
            DARBS_TRY(reserve(ctx, ctx->grad_image, sizeof(float) * 3 * px));
            d_lgrad = (float*)ctx->grad_image.ptr;
        }
        DARBS_TRY(launch_loss(ctx, width, height, d_image, d_target, lambda, d_lgrad, d_sums));
        d_gimg = d_lgrad;
        if (staged >= 0) {  // the slot's last reader: a later prefetch into it waits for this
            DARBS_CUDA_TRY(ctx, cudaEventRecord(ctx->target_read[staged], ctx->stream));
            ctx->target_read_pending[staged] = true;
        }
    }
    if (param_grads) {
        {
            StageScope ts(ctx, ST_RENDER_BWD);
            DARBS_TRY(launch_render_bwd(ctx, kp, width, height, background, d_gimg,
                                        (const float*)ctx->t_final.ptr, (const int32_t*)ctx->processed.ptr, n));
        }
        {
            StageScope ts(ctx, ST_PREPROCESS_BWD);
            DARBS_TRY(launch_param_grads(ctx, psi, n, d_raw, cam, d_valid, (const float*)ctx->splat_grads.ptr,
                                         d_conic, d_pgrads, overwrite));
        }
    }
    DARBS_TRY(st.finish());
    DARBS_TRY(sti.finish());
    // flags (2 ints) and loss sums (3 doubles) travel to a pinned ring slot; the caller either waits
    // for them now (loss_out) or collects them later with darbs_cuda_pop_loss, so that a training
    // loop never has to drain the stream between two iterations
    // A view that is being captured into a CUDA graph (possible with darbs_cuda_set_entry_capacity:
    // nothing above synchronises with the host) reports neither loss nor status: the ring's events
    // cannot be waited for from inside a capture, and a replay has no call to return them from.
    {
        cudaStreamCaptureStatus capturing = cudaStreamCaptureStatusNone;
        DARBS_CUDA_TRY(ctx, cudaStreamIsCapturing(ctx->stream, &capturing));
        if (capturing != cudaStreamCaptureStatusNone) {
            if (loss_out) return fail(ctx, DARBS_CONTRACT_VIOLATION, "evaluate_view: loss_out inside a stream capture");
            return DARBS_OK;
        }
    }
    if (ctx->loss_pending == kLossRing) {  // nobody collects them: forget the oldest
        ctx->loss_head = (ctx->loss_head + 1) % kLossRing;
        --ctx->loss_pending;
    }
    LossSlot& slot = ctx->loss_ring[(ctx->loss_head + ctx->loss_pending) % kLossRing];
    slot.count = target ? (double)(3 * px) : 0.0;
    slot.lambda = lambda;
    slot.fixed_point = ctx->deterministic != 0;
    DARBS_CUDA_TRY(ctx, cudaMemcpyAsync(slot.host, d_flags, 40, cudaMemcpyDeviceToHost, ctx->stream));
    DARBS_CUDA_TRY(ctx, cudaEventRecord(slot.done, ctx->stream));
    ++ctx->loss_pending;
    if (loss_out) {
        // the synchronous form: drain older pending losses, then this one
        darbs_status st_last = DARBS_OK;
        while (ctx->loss_pending > 0) st_last = darbs_cuda_pop_loss(ctx, loss_out);
        return st_last;
    }
    return DARBS_OK;
}

darbs_status darbs_cuda_set_entry_capacity(darbs_cuda_ctx* ctx, int64_t entries) {
    CTX_OR_FAIL(ctx);
    if (entries < 0 || entries >= ((int64_t)1 << 30))
        return fail(ctx, DARBS_INVALID_PARAMETER, "set_entry_capacity: negative or 2^30 and more");
    ctx->entry_capacity = entries;
    return DARBS_OK;
}

darbs_status darbs_cuda_set_cull_segment(darbs_cuda_ctx* ctx, int entries) {
    CTX_OR_FAIL(ctx);
    if (entries < 0) return fail(ctx, DARBS_INVALID_PARAMETER, "set_cull_segment: negative");
    ctx->cull_segment = entries;
    return DARBS_OK;
}

darbs_status darbs_cuda_set_deterministic(darbs_cuda_ctx* ctx, int enabled) {
    CTX_OR_FAIL(ctx);
    ctx->deterministic = enabled ? 1 : 0;
    return DARBS_OK;
}

darbs_status darbs_cuda_set_accumulate(darbs_cuda_ctx* ctx, int accumulate) {
    CTX_OR_FAIL(ctx);
    ctx->accumulate = accumulate ? 1 : 0;
    return DARBS_OK;
}

darbs_status darbs_cuda_prefetch_target(darbs_cuda_ctx* ctx, const float* host_image, int64_t count) {
    CTX_OR_FAIL(ctx);
    if (!host_image || count <= 0) return fail(ctx, DARBS_INVALID_PARAMETER, "prefetch_target: empty image");
    DeviceGuard guard(ctx->device);
    const int slot = ctx->target_next;
    ctx->target_next ^= 1;
    ctx->target_src[slot] = nullptr;
    DARBS_TRY(reserve(ctx, ctx->target_stage[slot], sizeof(float) * (size_t)count));
    // behind the cull of the last view queued (its forward and backward kernels hide the transfer);
    // that point is also past every reader of this slot, used two views ago
    if (ctx->have_after_cull) {
        DARBS_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->copy_stream, ctx->after_cull, 0));
    } else {
        DARBS_CUDA_TRY(ctx, cudaEventRecord(ctx->copy_begin, ctx->stream));
        DARBS_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->copy_stream, ctx->copy_begin, 0));
    }
    if (ctx->target_read_pending[slot]) {  // the loss kernels that read the slot's previous image
        DARBS_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->copy_stream, ctx->target_read[slot], 0));
        ctx->target_read_pending[slot] = false;
    }
    DARBS_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->target_stage[slot].ptr, host_image, sizeof(float) * (size_t)count,
                                        cudaMemcpyHostToDevice, ctx->copy_stream));
    DARBS_CUDA_TRY(ctx, cudaEventRecord(ctx->target_done[slot], ctx->copy_stream));
    ctx->target_src[slot] = host_image;
    return DARBS_OK;
}

darbs_status darbs_cuda_pop_loss(darbs_cuda_ctx* ctx, double loss_out[4]) {
    CTX_OR_FAIL(ctx);
    if (ctx->loss_pending == 0) return fail(ctx, DARBS_CONTRACT_VIOLATION, "pop_loss: no evaluate_view pending");
    DeviceGuard guard(ctx->device);
    LossSlot& slot = ctx->loss_ring[ctx->loss_head];
    ctx->loss_head = (ctx->loss_head + 1) % kLossRing;
    --ctx->loss_pending;
    DARBS_CUDA_TRY(ctx, cudaEventSynchronize(slot.done));
    const int* flags = (const int*)slot.host;
    double sums[3];
    read_loss_sums((const char*)slot.host + 16, slot.fixed_point, sums);
    double out[4] = {0.0, 0.0, 0.0, 0.0};
    if (slot.count > 0.0) {
        out[1] = sums[0] / slot.count;                                   // l1      loss.cpp:188
        out[2] = 0.5 * sums[2] / slot.count;                             // dssim   loss.cpp:226-227 (sum of 1 - SSIM)
        out[0] = (1.0 - slot.lambda) * out[1] + slot.lambda * out[2];    // total   loss.cpp:228
        out[3] = sums[1] / slot.count;                                   // mse     image.cpp mse()
    }
    if (loss_out)
        for (int i = 0; i < 4; ++i) loss_out[i] = out[i];
    unsigned long long overflow;
    std::memcpy(&overflow, (const char*)slot.host + 8, 8);
    if (overflow)
        return fail(ctx, DARBS_CONTRACT_VIOLATION,
                    "evaluate_view: more tile entries than darbs_cuda_set_entry_capacity promised; the view is incomplete");
    if (flags[0] & 1) return fail(ctx, DARBS_INVALID_PARAMETER, "covariance_from_scale_rot: scale must be positive");
    if (flags[0] & 2) return fail(ctx, DARBS_NUMERIC_ERROR, "conic_and_radius: covariance not positive definite");
    if (flags[1] == 0) return fail(ctx, DARBS_NUMERIC_ERROR, "fit_scene: all primitives culled in one view");
    if (slot.count > 0.0 && !std::isfinite(out[0])) return fail(ctx, DARBS_NUMERIC_ERROR, "fit_scene: loss diverged");
    return DARBS_OK;
}

darbs_status darbs_cuda_loss_total(darbs_cuda_ctx* ctx, int width, int height, const float* rendered,
                                   const float* target, double lambda, double loss_out[4],
                                   float* grad_image, darbs_space space) {
    CTX_OR_FAIL(ctx);
    if (width < 0 || height < 0) return fail(ctx, DARBS_INVALID_PARAMETER, "loss_total: negative size");
    const size_t px = (size_t)width * height;
    if (px > 0 && (!rendered || !target)) return fail(ctx, DARBS_INVALID_PARAMETER, "loss_total: image is NULL");
    if (!(lambda >= 0.0 && lambda <= 1.0)) return fail(ctx, DARBS_INVALID_PARAMETER, "lambda must lie in [0, 1]");
    DeviceGuard guard(ctx->device);
    reset_stage_marks(ctx, {ST_LOSS});
    Stager st(ctx, space);
    const float *d_img, *d_tgt;
    float* d_grad;
    DARBS_TRY(st.in(rendered, 3 * px, &d_img));
    DARBS_TRY(st.in(target, 3 * px, &d_tgt));
    DARBS_TRY(st.out(grad_image, 3 * px, &d_grad));
    double* d_sums = (double*)((unsigned long long*)ctx->counters.ptr + 14);
    {
        StageScope ts(ctx, ST_LOSS);
        DARBS_TRY(launch_loss(ctx, width, height, d_img, d_tgt, lambda, d_grad, d_sums));
    }
    DARBS_TRY(st.finish());
    if (loss_out) {
        DARBS_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->pinned, d_sums, sizeof(double) * 3, cudaMemcpyDeviceToHost,
                                            ctx->stream));
        DARBS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
        double sums[3];
        read_loss_sums(ctx->pinned, ctx->deterministic != 0, sums);
        const double count = (double)(3 * px);
        loss_out[1] = px ? sums[0] / count : 0.0;                      // loss.cpp:188
        loss_out[2] = px ? 0.5 * sums[2] / count : 0.0;                // loss.cpp:226-227 (sum of 1 - SSIM)
        loss_out[0] = (1.0 - lambda) * loss_out[1] + lambda * loss_out[2];
        loss_out[3] = px ? sums[1] / count : 0.0;
    }
    return DARBS_OK;
}

darbs_status darbs_cuda_adam_step(darbs_cuda_ctx* ctx, int64_t dim, float* params, const float* grads,
                                  float* m, float* v, const float* lrs, int t, darbs_space space) {
    CTX_OR_FAIL(ctx);
    if (dim < 0 || t < 1) return fail(ctx, DARBS_INVALID_PARAMETER, "adam_step: bad dim or step");
    if (dim > 0 && (!params || !grads || !m || !v || !lrs))
        return fail(ctx, DARBS_CONTRACT_VIOLATION, "adam_step: shape mismatch");  // optim.hpp:26-29
    DeviceGuard guard(ctx->device);
    reset_stage_marks(ctx, {ST_ADAM});
    Stager st(ctx, space);
    float *d_p, *d_m, *d_v;
    const float *d_g, *d_lr;
    DARBS_TRY(st.inout(params, (size_t)dim, &d_p));
    DARBS_TRY(st.inout(m, (size_t)dim, &d_m));
    DARBS_TRY(st.inout(v, (size_t)dim, &d_v));
    DARBS_TRY(st.in(grads, (size_t)dim, &d_g));
    DARBS_TRY(st.in(lrs, (size_t)dim, &d_lr));
    {
        StageScope ts(ctx, ST_ADAM);
        DARBS_TRY(launch_adam(ctx, dim, d_p, d_g, d_m, d_v, d_lr, t));
    }
    return st.finish();
}

// ---- instrumentation --------------------------------------------------------------

darbs_status darbs_cuda_set_stage_timing(darbs_cuda_ctx* ctx, int enabled) {
    CTX_OR_FAIL(ctx);
    ctx->timing = enabled ? 1 : 0;
    for (int s = 0; s < 8; ++s) ctx->stage_ms[s] = -1.0;
    return DARBS_OK;
}

darbs_status darbs_cuda_stage_times(darbs_cuda_ctx* ctx, double out_ms[8]) {
    CTX_OR_FAIL(ctx);
    DeviceGuard guard(ctx->device);
    DARBS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    for (int s = 0; s < 8; ++s) {
        if (ctx->stage_ms[s] == -2.0) {
            float ms = 0.f;
            cudaError_t e = cudaEventElapsedTime(&ms, ctx->timer.ev[2 * s], ctx->timer.ev[2 * s + 1]);
            ctx->stage_ms[s] = e == cudaSuccess ? (double)ms : -1.0;
        }
        out_ms[s] = ctx->stage_ms[s] < 0.0 ? 0.0 : ctx->stage_ms[s];
    }
    return DARBS_OK;
}

darbs_status darbs_cuda_work_counters(darbs_cuda_ctx* ctx, int64_t out[8]) {
    CTX_OR_FAIL(ctx);
    if (!ctx->have_forward) return fail(ctx, DARBS_CONTRACT_VIOLATION, "no forward on this context yet");
    DeviceGuard guard(ctx->device);
    const size_t px = (size_t)ctx->fwd_w * ctx->fwd_h;
    unsigned long long* c = (unsigned long long*)ctx->counters.ptr;
    DARBS_CUDA_TRY(ctx, cudaMemsetAsync(c + 1, 0, sizeof(unsigned long long) * 2, ctx->stream));
    if (ctx->fwd_contrib)
        DARBS_TRY(launch_sum_counts(ctx, (int64_t)px, (const int32_t*)ctx->processed.ptr, ctx->fwd_contrib));
    DARBS_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->pinned, c, sizeof(unsigned long long) * 8,
                                        cudaMemcpyDeviceToHost, ctx->stream));
    DARBS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    unsigned long long total = 0;  // K as the device counted it (the host may only know a capacity)
    DARBS_CUDA_TRY(ctx, cudaMemcpy(&total, c + 8, sizeof(total), cudaMemcpyDeviceToHost));
    for (int i = 0; i < 8; ++i) out[i] = (int64_t)((unsigned long long*)ctx->pinned)[i];
    out[0] = (int64_t)total;
    return DARBS_OK;
}

}  // extern "C"
