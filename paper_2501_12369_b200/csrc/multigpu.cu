// multigpu.cu — view-parallel training iteration behind the C ABI.
//
// fit_scene's iteration (reference src/fit3d.cpp:104-184) walks the views serially and meets only
// at `grads[owner] += ...` (:148-158).  Here every rank (one process per GPU) holds a replica of
// the 14 N raw parameters and the Adam state, evaluates ITS views (view v belongs to rank
// v mod world) into one 14 N float32 gradient buffer, and ONE all-reduce (ncclSum, no 1/V scaling)
// over NVLink makes the buffers equal before the replicated Adam step; the reported loss is the
// view mean (fit3d.cpp:161-165), a second all-reduce of four doubles.  The all-reduce runs on its
// own stream in kChunks pieces, and Adam updates piece c while piece c + 1 is still being reduced.
//
// NCCL is bound at run time (dlopen of libnccl.so.2; DARBS_NCCL_LIB overrides the name): the
// single-GPU library has no link-time dependency on it, and a process that already loaded torch's
// bundled NCCL shares that copy.
#include <dlfcn.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace darbs_b200 {

// the subset of nccl.h this file needs (NCCL 2.x ABI: nccl.h:37-41, :146-181, :260-286, :392)
struct NcclId {
    char internal[128];
};
using NcclComm = void*;
enum { kNcclSum = 0, kNcclFloat32 = 7, kNcclFloat64 = 8 };

struct NcclApi {
    void* lib = nullptr;
    int (*GetUniqueId)(NcclId*) = nullptr;
    int (*CommInitRank)(NcclComm*, int, NcclId, int) = nullptr;
    int (*CommDestroy)(NcclComm) = nullptr;
    int (*AllReduce)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(int) = nullptr;
};

static NcclApi* nccl_api(std::string* why) {
    static NcclApi api;
    static bool tried = false;
    static std::string error;
    if (!tried) {
        tried = true;
        const char* names[] = {std::getenv("DARBS_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
        for (const char* nm : names) {
            if (!nm || !*nm) continue;
            api.lib = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
            if (api.lib) break;
            error = dlerror();
        }
        if (api.lib) {
            api.GetUniqueId = (int (*)(NcclId*))dlsym(api.lib, "ncclGetUniqueId");
            api.CommInitRank = (int (*)(NcclComm*, int, NcclId, int))dlsym(api.lib, "ncclCommInitRank");
            api.CommDestroy = (int (*)(NcclComm))dlsym(api.lib, "ncclCommDestroy");
            api.AllReduce = (int (*)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t))dlsym(api.lib, "ncclAllReduce");
            api.GetErrorString = (const char* (*)(int))dlsym(api.lib, "ncclGetErrorString");
            if (!api.GetUniqueId || !api.CommInitRank || !api.CommDestroy || !api.AllReduce) {
                error = "libnccl lacks ncclGetUniqueId / ncclCommInitRank / ncclCommDestroy / ncclAllReduce";
                api.lib = nullptr;
            }
        }
    }
    if (!api.lib) {
        if (why) *why = error;
        return nullptr;
    }
    return &api;
}

struct Comm {  // owned by the context (ctx->comm)
    NcclComm comm = nullptr;
    int rank = 0, world = 1;
    cudaStream_t stream = nullptr;             // the all-reduce runs here
    cudaEvent_t grads_ready = nullptr;         // main stream -> comm stream
    cudaEvent_t piece_done[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    double* d_loss = nullptr;                  // 4 doubles on the device
};
static constexpr int kChunks = 4;

static darbs_status nccl_fail(darbs_cuda_ctx* ctx, NcclApi* api, int rc, const char* what) {
    return fail(ctx, DARBS_CUDA_ERROR, std::string("NCCL: ") + what + ": " +
                                           (api && api->GetErrorString ? api->GetErrorString(rc) : "error " + std::to_string(rc)));
}

void destroy_comm(darbs_cuda_ctx* ctx) {
    Comm* c = (Comm*)ctx->comm;
    if (!c) return;
    NcclApi* api = nccl_api(nullptr);
    if (c->comm && api) api->CommDestroy(c->comm);
    if (c->stream) cudaStreamDestroy(c->stream);
    if (c->grads_ready) cudaEventDestroy(c->grads_ready);
    for (cudaEvent_t e : c->piece_done)
        if (e) cudaEventDestroy(e);
    if (c->d_loss) cudaFree(c->d_loss);
    delete c;
    ctx->comm = nullptr;
}

}  // namespace darbs_b200

using namespace darbs_b200;

extern "C" {

darbs_status darbs_cuda_comm_unique_id(darbs_comm_id* out) {
    if (!out) return fail(nullptr, DARBS_INVALID_PARAMETER, "comm_unique_id: out is NULL");
    std::string why;
    NcclApi* api = nccl_api(&why);
    if (!api) return fail(nullptr, DARBS_CUDA_ERROR, "NCCL is not available: " + why);
    static_assert(sizeof(darbs_comm_id) == sizeof(NcclId), "ncclUniqueId is 128 bytes");
    NcclId id;
    const int rc = api->GetUniqueId(&id);
    if (rc != 0) return nccl_fail(nullptr, api, rc, "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof(id));
    return DARBS_OK;
}

darbs_status darbs_cuda_comm_init(darbs_cuda_ctx* ctx, const darbs_comm_id* id, int rank, int world) {
    if (!ctx) return fail(nullptr, DARBS_INVALID_PARAMETER, "context is NULL");
    if (!id || world < 1 || rank < 0 || rank >= world) return fail(ctx, DARBS_INVALID_PARAMETER, "comm_init: bad rank / world");
    std::string why;
    NcclApi* api = nccl_api(&why);
    if (!api) return fail(ctx, DARBS_CUDA_ERROR, "NCCL is not available: " + why);
    destroy_comm(ctx);
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(ctx->device);
    Comm* c = new Comm();
    c->rank = rank;
    c->world = world;
    NcclId nid;
    std::memcpy(&nid, id, sizeof(nid));
    const int rc = api->CommInitRank(&c->comm, world, nid, rank);
    darbs_status st = DARBS_OK;
    if (rc != 0) {
        st = nccl_fail(ctx, api, rc, "ncclCommInitRank");
    } else if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
               cudaEventCreateWithFlags(&c->grads_ready, cudaEventDisableTiming) != cudaSuccess ||
               cudaMalloc(&c->d_loss, 4 * sizeof(double)) != cudaSuccess) {
        st = fail(ctx, DARBS_CUDA_ERROR, "comm_init: stream / event / buffer creation failed");
    } else {
        for (int i = 0; i < kChunks; ++i) cudaEventCreateWithFlags(&c->piece_done[i], cudaEventDisableTiming);
    }
    ctx->comm = c;
    if (st != DARBS_OK) destroy_comm(ctx);
    if (prev >= 0 && prev != ctx->device) cudaSetDevice(prev);
    return st;
}

darbs_status darbs_cuda_comm_destroy(darbs_cuda_ctx* ctx) {
    if (!ctx) return fail(nullptr, DARBS_INVALID_PARAMETER, "context is NULL");
    destroy_comm(ctx);
    return DARBS_OK;
}

darbs_status darbs_cuda_allreduce_adam_step(darbs_cuda_ctx* ctx, int64_t dim_, float* params, float* grads, float* m,
                                            float* v, const float* lrs, int t) {
    if (!ctx) return fail(nullptr, DARBS_INVALID_PARAMETER, "context is NULL");
    if (dim_ < 0 || t < 1) return fail(ctx, DARBS_INVALID_PARAMETER, "allreduce_adam_step: bad dim or step");
    if (dim_ > 0 && (!params || !grads || !m || !v || !lrs))
        return fail(ctx, DARBS_INVALID_PARAMETER, "allreduce_adam_step: NULL array");
    Comm* c = (Comm*)ctx->comm;
    const int world = c ? c->world : 1;
    const size_t dim = (size_t)dim_;
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != ctx->device) cudaSetDevice(ctx->device);
    struct Restore {
        int prev, dev;
        ~Restore() {
            if (prev >= 0 && prev != dev) cudaSetDevice(prev);
        }
    } restore{prev, ctx->device};
    std::string why;
    NcclApi* api = world > 1 ? nccl_api(&why) : nullptr;
    if (world > 1 && !api) return fail(ctx, DARBS_CUDA_ERROR, "NCCL is not available: " + why);
    if (world > 1) {
        DARBS_CUDA_TRY(ctx, cudaEventRecord(c->grads_ready, ctx->stream));
        DARBS_CUDA_TRY(ctx, cudaStreamWaitEvent(c->stream, c->grads_ready, 0));
    }
    const size_t piece = ((dim + kChunks - 1) / kChunks + 3) & ~(size_t)3;
    for (int i = 0; i < kChunks; ++i) {
        const size_t lo = (size_t)i * piece, hi = lo + piece < dim ? lo + piece : dim;
        if (lo >= hi) break;
        if (world > 1) {
            const int rc = api->AllReduce(grads + lo, grads + lo, hi - lo, kNcclFloat32, kNcclSum, c->comm, c->stream);
            if (rc != 0) return nccl_fail(ctx, api, rc, "ncclAllReduce");
            DARBS_CUDA_TRY(ctx, cudaEventRecord(c->piece_done[i], c->stream));
            DARBS_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, c->piece_done[i], 0));
        }
        DARBS_TRY(launch_adam(ctx, (int64_t)(hi - lo), params + lo, grads + lo, m + lo, v + lo, lrs + lo, t));
    }
    return DARBS_OK;
}

darbs_status darbs_cuda_train_step(darbs_cuda_ctx* ctx, const darbs_kernel_spec* kernel, double psi, int64_t n,
                                   float* params, float* grads, float* m, float* v, const float* lrs,
                                   int n_local_views, const double* cameras, const float* const* targets,
                                   double lambda, const float background[3], int t, int n_views_total,
                                   double loss_out[4]) {
    if (!ctx) return fail(nullptr, DARBS_INVALID_PARAMETER, "context is NULL");
    if (n < 0 || n_local_views < 0 || t < 1 || n_views_total < 1)
        return fail(ctx, DARBS_INVALID_PARAMETER, "train_step: bad size, view count or step");
    if (n > 0 && (!params || !grads || !m || !v || !lrs)) return fail(ctx, DARBS_INVALID_PARAMETER, "train_step: NULL array");
    if (n_local_views > 0 && (!cameras || !targets)) return fail(ctx, DARBS_INVALID_PARAMETER, "train_step: NULL views");
    Comm* c = (Comm*)ctx->comm;
    const int world = c ? c->world : 1;
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != ctx->device) cudaSetDevice(ctx->device);
    struct Restore {
        int prev, dev;
        ~Restore() {
            if (prev >= 0 && prev != dev) cudaSetDevice(prev);
        }
    } restore{prev, ctx->device};
    const size_t dim = (size_t)n * DARBS_PARAMS_PER_PRIMITIVE;

    // this rank's views (fit3d.cpp:108-159); the first one overwrites the gradient buffer
    double sums[4] = {0.0, 0.0, 0.0, 0.0};
    darbs_status view_status = DARBS_OK;
    if (n_local_views == 0 && dim)
        DARBS_CUDA_TRY(ctx, cudaMemsetAsync(grads, 0, sizeof(float) * dim, ctx->stream));
    int pending = 0;
    auto collect = [&]() {
        double one[4];
        const darbs_status st = darbs_cuda_pop_loss(ctx, one);
        if (st != DARBS_OK && view_status == DARBS_OK) view_status = st;
        for (int i = 0; i < 4; ++i) sums[i] += one[i];
        --pending;
    };
    for (int view = 0; view < n_local_views; ++view) {
        if (view == 0) DARBS_TRY(darbs_cuda_set_accumulate(ctx, 0));
        const darbs_status st = darbs_cuda_evaluate_view(ctx, kernel, psi, n, params, cameras + (size_t)view * DARBS_CAMERA_DOUBLES,
                                                         background, targets[view], lambda, nullptr, grads, nullptr, nullptr,
                                                         DARBS_DEVICE, DARBS_DEVICE);
        if (st != DARBS_OK) {  // leave the context clean for the next caller: no pending loss, "+=" mode
            while (pending > 0) collect();
            darbs_cuda_set_accumulate(ctx, 1);
            return st;
        }
        ++pending;
        if (pending > 2) collect();  // losses are collected two views late: the stream never drains
    }

    // gradients summed over all ranks' views, in kChunks pieces; Adam follows piece by piece
    {
        const darbs_status st = darbs_cuda_allreduce_adam_step(ctx, (int64_t)dim, params, grads, m, v, lrs, t);
        if (st != DARBS_OK) {
            while (pending > 0) collect();
            return st;
        }
    }
    NcclApi* api = world > 1 ? nccl_api(nullptr) : nullptr;
    while (pending > 0) collect();
    if (view_status != DARBS_OK) return view_status;

    if (loss_out) {  // the view mean over ALL views (fit3d.cpp:161-165)
        if (world > 1) {
            DARBS_CUDA_TRY(ctx, cudaMemcpyAsync(c->d_loss, sums, sizeof(sums), cudaMemcpyHostToDevice, c->stream));
            const int rc = api->AllReduce(c->d_loss, c->d_loss, 4, kNcclFloat64, kNcclSum, c->comm, c->stream);
            if (rc != 0) return nccl_fail(ctx, api, rc, "ncclAllReduce (loss)");
            DARBS_CUDA_TRY(ctx, cudaMemcpyAsync(sums, c->d_loss, sizeof(sums), cudaMemcpyDeviceToHost, c->stream));
            DARBS_CUDA_TRY(ctx, cudaStreamSynchronize(c->stream));
        }
        for (int i = 0; i < 4; ++i) loss_out[i] = sums[i] / (double)n_views_total;
        if (!std::isfinite(loss_out[0])) return fail(ctx, DARBS_NUMERIC_ERROR, "fit_scene: loss diverged");
    }
    return DARBS_OK;
}

}  // extern "C"
