#include <cstdio>
__global__ void k(float* out) {
    float x = 1.0f + 0.0f * threadIdx.x, y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    out[0] = y;
    float z; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(z) : "f"(x - 1.0f)); out[1] = z;
}
int main() { float* d; cudaMalloc(&d, 8); k<<<1, 1>>>(d); float h[2]; cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  printf("rcp(1)=%.9g bits %08x ex2(0)=%.9g\n", h[0], *(unsigned*)&h[0], h[1]); }
