// Stand-alone check and timing of csrc/radix.cuh on one B200:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2501_12369_b200/csrc -o scratch/sort/sort_bench scratch/sort/sort_bench.cu
// Sorts random pairs, compares with std::stable_sort, prints microseconds per sort.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <vector>

#define DARBS_RADIX_PROFILE
#include "radix.cuh"

using namespace darbs_b200::radix;

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            std::exit(1);                                                              \
        }                                                                              \
    } while (0)

template <typename KeyT>
int run(const char* name, unsigned n, Plan plan, unsigned key_mask, int reps) {
    std::mt19937_64 rng(n * 7 + plan.passes);
    std::vector<KeyT> keys(n);
    std::vector<unsigned> vals(n);
    for (unsigned i = 0; i < n; ++i) {
        keys[i] = (KeyT)(rng() & key_mask);
        vals[i] = i;
    }
    if (n > 100) {  // duplicates and runs
        for (unsigned i = 0; i < n / 10; ++i) keys[i] = keys[0];
    }
    KeyT *k0, *k1;
    unsigned *v0, *v1, *ws;
    const size_t words = workspace_words(n, plan.passes);
    CK(cudaMalloc(&k0, sizeof(KeyT) * (n + 16)));
    CK(cudaMalloc(&k1, sizeof(KeyT) * (n + 16)));
    CK(cudaMalloc(&v0, 4 * (size_t)(n + 16)));
    CK(cudaMalloc(&v1, 4 * (size_t)(n + 16)));
    CK(cudaMalloc(&ws, 4 * words));
    cudaStream_t s;
    CK(cudaStreamCreate(&s));
    cudaEvent_t e0, e1, e2;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventCreate(&e2));
    float best = 1e9f, best_h = 1e9f;
    for (int r = 0; r < reps; ++r) {
        CK(cudaMemcpyAsync(k0, keys.data(), sizeof(KeyT) * n, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(v0, vals.data(), 4 * (size_t)n, cudaMemcpyHostToDevice, s));
        CK(cudaMemsetAsync(ws, 0, 4 * words, s));
        CK(cudaEventRecord(e0, s));
        CK(launch_histogram<KeyT>(k0, n, plan, ws + kHistAt, 148, s));
        CK(cudaEventRecord(e1, s));
        CK(launch_passes<KeyT>(k0, v0, k1, v1, n, plan, ws, ws + kHistAt, ws + kStatusAt, s));
        CK(cudaEventRecord(e2, s));
        CK(cudaStreamSynchronize(s));
        float ms, mh;
        CK(cudaEventElapsedTime(&mh, e0, e1));
        CK(cudaEventElapsedTime(&ms, e1, e2));
        best = std::min(best, ms);
        best_h = std::min(best_h, mh);
    }
    {
        long long prof[16];
        CK(cudaMemcpy(prof, g_prof, sizeof(prof), cudaMemcpyDeviceToHost));
        std::printf("   first chunk cycles:");
        for (int i = 1; i < 7; ++i) std::printf(" %lld", prof[i]);
        std::printf("   last chunk:");
        for (int i = 1; i < 7; ++i) std::printf(" %lld", prof[8 + i]);
        std::printf("\n");
    }
    std::vector<KeyT> out_k(n);
    std::vector<unsigned> out_v(n);
    const bool odd = plan.passes & 1;
    CK(cudaMemcpy(out_k.data(), odd ? k1 : k0, sizeof(KeyT) * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(out_v.data(), odd ? v1 : v0, 4 * (size_t)n, cudaMemcpyDeviceToHost));
    std::vector<unsigned> order(n);
    std::iota(order.begin(), order.end(), 0u);
    unsigned sort_mask = 0;
    for (int p = 0; p < plan.passes; ++p) sort_mask |= ((1u << plan.bits[p]) - 1u) << plan.shift[p];
    std::stable_sort(order.begin(), order.end(),
                     [&](unsigned a, unsigned b) { return (keys[a] & sort_mask) < (keys[b] & sort_mask); });
    size_t bad = 0;
    for (unsigned i = 0; i < n; ++i)
        if (out_v[i] != order[i] || out_k[i] != keys[order[i]]) ++bad;
    std::printf("%-28s n=%9u passes=%d  histogram %7.1f us  passes %7.1f us (%.1f us/pass, %.0f GB/s per pass)  %s\n", name, n,
                plan.passes, best_h * 1e3f, best * 1e3f, best * 1e3f / plan.passes,
                2.0 * n * (sizeof(KeyT) + 4) / (best * 1e-3 / plan.passes) / 1e9, bad ? "MISMATCH" : "ok");
    cudaFree(k0); cudaFree(k1); cudaFree(v0); cudaFree(v1); cudaFree(ws);
    return bad != 0;
}

int main() {
    int fails = 0;
    CK(cudaMalloc(&g_prof, 16 * sizeof(long long)));
    CK(cudaMemset(g_prof, 0, 16 * sizeof(long long)));
    const Plan depth{4, {0, 8, 16, 24}, {8, 8, 8, 8}};
    const Plan tile13{2, {0, 8}, {7, 7}};
    const Plan tile16{2, {0, 8}, {8, 8}};
    const Plan one{1, {0}, {8}};
    const Plan tile3{3, {0, 8, 16}, {8, 1, 8}};
    for (unsigned n : {1u, 31u, 8192u, 8193u, 100000u}) fails += run<unsigned>("u32 depth keys", n, depth, 0xffffffffu, 2);
    fails += run<unsigned short>("u16 tile keys small", 12345, tile16, 0xffffu, 2);
    fails += run<unsigned>("u32 split digits", 777777, tile3, 0x00ff01ffu, 2);
    fails += run<unsigned>("u32 one pass", 3000000, one, 0xffu, 3);
    fails += run<unsigned>("u32 depth keys", 1000000, depth, 0xffffffffu, 10);
    fails += run<unsigned>("u32 depth keys", 3000000, depth, 0xffffffffu, 5);
    fails += run<unsigned short>("u16 tile keys (7+7 bits)", 4200000, tile13, 0x7f7fu, 10);
    fails += run<unsigned short>("u16 tile keys (8+8 bits)", 4200000, tile16, 0xffffu, 10);
    fails += run<unsigned short>("u16 tile keys (8+8 bits)", 17000000, tile16, 0xffffu, 5);
    fails += run<unsigned short>("u16 tile keys (8+8 bits)", 50000000, tile16, 0xffffu, 3);
    std::printf(fails ? "FAILED\n" : "all sorts ok\n");
    return fails;
}
