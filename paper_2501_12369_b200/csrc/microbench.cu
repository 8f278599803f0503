// microbench.cu — register-only micro-benchmarks of the FP32 FMA pipe and the
// MUFU (special-function) pipe.  The render kernels are bound by the issue rate
// of these two pipes, not by HBM or tensor cores, and MEASURED_PEAKS.json has no
// entry for them (SURVEY.md §8d asks the build to measure them on the box).
#include "common.cuh"

namespace darbs_b200 {
namespace {

constexpr int kIters = 4096;

// 8 independent FMA chains per thread: no dependency stalls at 4-cycle latency
// with >= 8 warps per scheduler.
// IMM = true lets ptxas use the immediate-operand FFMA form; IMM = false keeps
// both multiplier and addend in registers (the form the render kernels issue).
template <bool IMM>
__global__ void __launch_bounds__(1024) ffma_kernel(float seed, float* sink, long long* cycles) {
    float a0 = seed + threadIdx.x, a1 = a0 + 1.f, a2 = a0 + 2.f, a3 = a0 + 3.f;
    float a4 = a0 + 4.f, a5 = a0 + 5.f, a6 = a0 + 6.f, a7 = a0 + 7.f;
    const float m = IMM ? 0.999f : 0.999f + (float)(blockIdx.x >> 30);
    const float c = IMM ? 0.001f : 0.001f + (float)(blockIdx.x >> 29);
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            a0 = fmaf(a0, m, c);
            a1 = fmaf(a1, m, c);
            a2 = fmaf(a2, m, c);
            a3 = fmaf(a3, m, c);
            a4 = fmaf(a4, m, c);
            a5 = fmaf(a5, m, c);
            a6 = fmaf(a6, m, c);
            a7 = fmaf(a7, m, c);
        }
    }
    long long t1 = clock64();
    float s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 12345.678f) sink[0] = s;  // keep the chains alive
    if (blockIdx.x == 0 && threadIdx.x == 0) cycles[0] = t1 - t0;
}

// Packed FP32 FMA (fma.rn.f32x2, FFMA2 in SASS): two FMAs per lane per instruction.
__global__ void __launch_bounds__(1024) ffma2_kernel(float seed, float* sink) {
    float2 a0 = make_float2(seed + threadIdx.x, seed + 0.5f), a1 = a0, a2 = a0, a3 = a0, a4 = a0, a5 = a0, a6 = a0,
           a7 = a0;
    a1.x += 1.f; a2.x += 2.f; a3.x += 3.f; a4.x += 4.f; a5.x += 5.f; a6.x += 6.f; a7.x += 7.f;
    const float mm = 0.999f + (float)(blockIdx.x >> 30), cc = 0.001f + (float)(blockIdx.x >> 29);
    const float2 m = make_float2(mm, mm), c = make_float2(cc, cc);
#pragma unroll 1
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            a0 = __ffma2_rn(a0, m, c);
            a1 = __ffma2_rn(a1, m, c);
            a2 = __ffma2_rn(a2, m, c);
            a3 = __ffma2_rn(a3, m, c);
            a4 = __ffma2_rn(a4, m, c);
            a5 = __ffma2_rn(a5, m, c);
            a6 = __ffma2_rn(a6, m, c);
            a7 = __ffma2_rn(a7, m, c);
        }
    }
    float s = a0.x + a1.x + a2.x + a3.x + a4.x + a5.x + a6.x + a7.x + a0.y + a1.y + a2.y + a3.y + a4.y + a5.y +
              a6.y + a7.y;
    if (s == 12345.678f) sink[0] = s;
}

__global__ void __launch_bounds__(1024) mufu_kernel(float seed, float* sink) {
    float a0 = seed + 1e-3f * threadIdx.x, a1 = a0 - 0.1f, a2 = a0 - 0.2f, a3 = a0 - 0.3f;
#pragma unroll 1
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a0));
            asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a1));
            asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a2));
            asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a3));
        }
    }
    float s = a0 + a1 + a2 + a3;
    if (s == 12345.678f) sink[0] = s;
}

// SM clock: one thread spins on a dependent FMA chain and reads the SM's cycle counter and the
// nanosecond global timer on both sides (the ratio is the clock the SM ran at; the earlier
// "one block's clock64 span over the kernel's event time" was wrong by the share of the kernel
// that block did not run for).
__global__ void clock_kernel(float seed, float* sink, long long* out) {
    unsigned long long g0, g1;
    float a = seed;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    const long long c0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 200000; ++i) a = fmaf(a, 0.999f, 0.001f);
    const long long c1 = clock64();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    if (a == 12345.678f) sink[0] = a;
    out[0] = c1 - c0;
    out[1] = (long long)(g1 - g0);
}

}  // namespace
}  // namespace darbs_b200

using namespace darbs_b200;

extern "C" darbs_status darbs_cuda_microbench(darbs_cuda_ctx* ctx, double out[8]) {
    if (!ctx) return fail(nullptr, DARBS_INVALID_PARAMETER, "context is NULL");
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != ctx->device) cudaSetDevice(ctx->device);
    cudaDeviceProp prop;
    DARBS_CUDA_TRY(ctx, cudaGetDeviceProperties(&prop, ctx->device));
    const int sms = prop.multiProcessorCount;
    const int blocks = sms * 2, threads = 1024;  // 2 x 1024 threads = full occupancy
    float* sink = (float*)((unsigned long long*)ctx->counters.ptr + 20);
    long long* cycles = (long long*)((unsigned long long*)ctx->counters.ptr + 22);
    cudaEvent_t e0 = ctx->timer.ev[14], e1 = ctx->timer.ev[15];
    float ms_f = 0.f, ms_m = 0.f, ms_i = 0.f, ms_2 = 0.f;
    for (int rep = 0; rep < 3; ++rep) {
        DARBS_CUDA_TRY(ctx, cudaEventRecord(e0, ctx->stream));
        ffma2_kernel<<<blocks, threads, 0, ctx->stream>>>(1.0f, sink);
        DARBS_CUDA_TRY(ctx, cudaEventRecord(e1, ctx->stream));
        DARBS_CUDA_TRY(ctx, cudaEventSynchronize(e1));
        DARBS_CUDA_TRY(ctx, cudaEventElapsedTime(&ms_2, e0, e1));
    }
    for (int rep = 0; rep < 3; ++rep) {
        DARBS_CUDA_TRY(ctx, cudaEventRecord(e0, ctx->stream));
        ffma_kernel<true><<<blocks, threads, 0, ctx->stream>>>(1.0f, sink, cycles);
        DARBS_CUDA_TRY(ctx, cudaEventRecord(e1, ctx->stream));
        DARBS_CUDA_TRY(ctx, cudaEventSynchronize(e1));
        DARBS_CUDA_TRY(ctx, cudaEventElapsedTime(&ms_i, e0, e1));
    }
    for (int rep = 0; rep < 3; ++rep) {  // last repetition counts (clocks ramped up)
        DARBS_CUDA_TRY(ctx, cudaEventRecord(e0, ctx->stream));
        ffma_kernel<false><<<blocks, threads, 0, ctx->stream>>>(1.0f, sink, cycles);
        DARBS_CUDA_TRY(ctx, cudaEventRecord(e1, ctx->stream));
        DARBS_CUDA_TRY(ctx, cudaEventSynchronize(e1));
        DARBS_CUDA_TRY(ctx, cudaEventElapsedTime(&ms_f, e0, e1));
    }
    for (int rep = 0; rep < 3; ++rep) {
        DARBS_CUDA_TRY(ctx, cudaEventRecord(e0, ctx->stream));
        mufu_kernel<<<blocks, threads, 0, ctx->stream>>>(0.5f, sink);
        DARBS_CUDA_TRY(ctx, cudaEventRecord(e1, ctx->stream));
        DARBS_CUDA_TRY(ctx, cudaEventSynchronize(e1));
        DARBS_CUDA_TRY(ctx, cudaEventElapsedTime(&ms_m, e0, e1));
    }
    clock_kernel<<<1, 1, 0, ctx->stream>>>(1.0f, sink, cycles);  // right behind the load: boosted clocks
    DARBS_TRY(check_launch(ctx, "microbench", 13));
    long long cyc[2] = {0, 1};
    DARBS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    DARBS_CUDA_TRY(ctx, cudaMemcpy(cyc, cycles, sizeof(cyc), cudaMemcpyDeviceToHost));
    const double n_thr = (double)blocks * threads;
    out[0] = n_thr * kIters * 32.0 / (ms_f * 1e-3);
    out[1] = n_thr * kIters * 16.0 / (ms_m * 1e-3);
    out[2] = cyc[1] > 0 ? 1e3 * (double)cyc[0] / (double)cyc[1] : 0.0;  // cycles per ns -> MHz
    out[3] = (double)sms;
    out[4] = n_thr * kIters * 32.0 / (ms_i * 1e-3);
    out[5] = n_thr * kIters * 32.0 / (ms_2 * 1e-3);  // packed instructions per second (x4 = FLOP/s)
    out[6] = out[7] = 0.0;
    if (prev >= 0 && prev != ctx->device) cudaSetDevice(prev);
    return DARBS_OK;
}
