// shared-memory atomic throughput on sm_100a: per-warp 256-word tables, random / constant digits
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(unsigned* out, int iters, unsigned seed) {
    __shared__ unsigned tab[32 * 256];
    for (int i = threadIdx.x; i < 32 * 256; i += blockDim.x) tab[i] = 0;
    __syncthreads();
    unsigned* t = tab + (threadIdx.x >> 5) * 256;
    const int lane = threadIdx.x & 31;
    unsigned x = threadIdx.x * 2654435761u + seed, acc = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        const unsigned d = (MODE & 1) ? 7u : (x >> 13) & 255u;
        if (MODE < 2) {  // peer mask through an atomic OR, read back, clear
            atomicOr(&t[d], 1u << lane);
            __syncwarp();
            const unsigned m = t[d];
            __syncwarp();
            t[d] = 0;
            __syncwarp();
            acc += m;
        } else if (MODE < 4) {  // atomicAdd with return
            acc += atomicAdd(&t[d], 1u);
        } else {  // plain LDS + STS
            const unsigned v = t[d];
            __syncwarp();
            t[d] = v + 1;
            __syncwarp();
            acc += v;
        }
        x = x * 1664525u + 1013904223u;
    }
    long long t1 = clock64();
    if (acc == 12345u) out[0] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) ((long long*)out)[1] = t1 - t0;
}
int main() {
    unsigned* d; cudaMalloc(&d, 64);
    const char* names[] = {"atomicOr+LDS+STS random", "atomicOr+LDS+STS same", "atomicAdd ret random", "atomicAdd ret same", "LDS+STS random", "LDS+STS same"};
    for (int warps : {4, 16, 32}) {
        for (int mode = 0; mode < 6; ++mode) {
            const int iters = 2000;
            for (int rep = 0; rep < 2; ++rep) {
                if (mode == 0) k<0><<<148, warps * 32>>>(d, iters, 1);
                if (mode == 1) k<1><<<148, warps * 32>>>(d, iters, 1);
                if (mode == 2) k<2><<<148, warps * 32>>>(d, iters, 1);
                if (mode == 3) k<3><<<148, warps * 32>>>(d, iters, 1);
                if (mode == 4) k<4><<<148, warps * 32>>>(d, iters, 1);
                if (mode == 5) k<5><<<148, warps * 32>>>(d, iters, 1);
                cudaDeviceSynchronize();
            }
            long long c[2]; cudaMemcpy(c, d, 16, cudaMemcpyDeviceToHost);
            std::printf("warps/SM %2d  %-26s %8.1f cycles per step per warp; %.1f SM-cycles per warp-step\n", warps, names[mode],
                        (double)c[1] / iters, (double)c[1] / iters / warps);
        }
    }
    return 0;
}
