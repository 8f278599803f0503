// broadcast shared-memory load cost per width: all lanes of a warp read the same address
#include <cstdio>
#include <cuda_runtime.h>
template <int W>
__global__ void k(float* out, int iters, int stride) {
    __shared__ __align__(16) float buf[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = i * 0.001f;
    __syncthreads();
    float acc = 0.f;
    int off = (blockIdx.x * 4) & 1023;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int a = (off + u * 4) & 2047;  // uniform across the warp, 16-byte aligned
            if (W == 32) { acc += buf[a]; }
            if (W == 64) { float2 v = *reinterpret_cast<const float2*>(buf + a); acc += v.x + v.y; }
            if (W == 128) { float4 v = *reinterpret_cast<const float4*>(buf + a); acc += v.x + v.y + v.z + v.w; }
        }
        off = (off + stride) & 1023;
    }
    if (acc == 12345.678f) out[0] = acc;
}
template <int W> void run(const char* name) {
    float* d; cudaMalloc(&d, 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 4096, grid = 148 * 8, block = 256;
    k<W><<<grid, block>>>(d, iters, 64); cudaDeviceSynchronize();
    cudaEventRecord(a); k<W><<<grid, block>>>(d, iters, 64); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double loads = (double)grid * (block / 32) * iters * 16;  // warp-level load instructions
    double cyc_per_load_sm = ms * 1e-3 * 1.965e9 * 148 / loads;
    printf("%s: %.3f ms, %.2f SM-cycles per warp-load\n", name, ms, cyc_per_load_sm);
}
int main() { run<32>("LDS.32 broadcast"); run<64>("LDS.64 broadcast"); run<128>("LDS.128 broadcast"); }
