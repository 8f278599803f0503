// VOTE / MATCH / LDS-STS chain throughput on sm_100a (one CTA per SM, W warps)
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(unsigned* out, int iters, unsigned seed) {
    __shared__ unsigned sm[32 * 256];
    unsigned x = threadIdx.x * 2654435761u + seed, acc = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (MODE == 0) {  // 8 independent ballots
#pragma unroll
            for (int b = 0; b < 8; ++b) acc += __ballot_sync(0xffffffffu, (x >> b) & 1u);
        } else if (MODE == 1) {  // match.any on 8-bit random values
            acc += __match_any_sync(0xffffffffu, x & 255u);
        } else if (MODE == 2) {  // popc + lop chain only
#pragma unroll
            for (int b = 0; b < 8; ++b) acc += __popc(x >> b);
        } else if (MODE == 3) {  // shfl
#pragma unroll
            for (int b = 0; b < 8; ++b) acc += __shfl_xor_sync(0xffffffffu, x, b + 1);
        } else if (MODE == 4) {  // reduce
#pragma unroll
            for (int b = 0; b < 8; ++b) acc += __reduce_add_sync(0xffffffffu, (x >> b) & 1u);
        }
        x = x * 1664525u + 1013904223u;
    }
    long long t1 = clock64();
    if (acc == 12345u) out[0] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) ((long long*)out)[1] = t1 - t0;
    (void)sm;
}
int main() {
    unsigned* d; cudaMalloc(&d, 64);
    const char* names[] = {"8 ballots", "match.any 8-bit", "8 popc", "8 shfl", "8 redux"};
    for (int warps : {1, 4, 16, 32}) {
        for (int mode = 0; mode < 5; ++mode) {
            const int iters = 2000;
            for (int rep = 0; rep < 2; ++rep) {
                if (mode == 0) k<0><<<148, warps * 32>>>(d, iters, 1);
                if (mode == 1) k<1><<<148, warps * 32>>>(d, iters, 1);
                if (mode == 2) k<2><<<148, warps * 32>>>(d, iters, 1);
                if (mode == 3) k<3><<<148, warps * 32>>>(d, iters, 1);
                if (mode == 4) k<4><<<148, warps * 32>>>(d, iters, 1);
                cudaDeviceSynchronize();
            }
            long long c[2]; cudaMemcpy(c, d, 16, cudaMemcpyDeviceToHost);
            std::printf("warps/SM %2d  %-16s %8.1f cycles per iteration per warp; %.2f cycles per op per SMSP\n", warps, names[mode],
                        (double)c[1] / iters, (double)c[1] / iters / (mode == 1 ? 1 : 8) / ((warps + 3) / 4));
        }
    }
    return 0;
}
