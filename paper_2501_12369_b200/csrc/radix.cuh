// radix.cuh — hand-written stable LSD radix sort for sm_100a, the sort under bin_splats
// (reference src/rasterizer.cpp:25-53: global stable depth order, then per-tile lists).
//
// One pass = ONE read and ONE write of the (key, value) pairs ("onesweep"): a CTA takes the next
// chunk of the input (ticket order), ranks its keys by the pass's digit with warp-private counters
// (peers found through a shared-memory table), publishes the chunk's digit histogram, finds the number of equal-digit
// keys in all earlier chunks by decoupled look-back over the published histograms (a window of
// predecessors per round trip), and scatters through shared memory so that every digit's keys
// leave as one contiguous run.  Stability: chunks are taken in input order, a warp's keys are
// contiguous, and ranks inside a (warp, digit) follow item-then-lane order.
//
// The digit histograms of the whole input are counted before the first pass (histogram_kernel for
// the depth keys; the tile keys' come out of the kernel that writes them, binning.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace darbs_b200 {
namespace radix {

constexpr int kBins = 256;  // digits are at most 8 bits wide
constexpr int kMaxPasses = 4;
constexpr unsigned kPartial = 1u << 30;    // status word: the chunk's own count
constexpr unsigned kInclusive = 2u << 30;  // status word: count of this and all earlier chunks
constexpr unsigned kValue = (1u << 30) - 1;
#ifndef DARBS_RADIX_LOOKBACK
#define DARBS_RADIX_LOOKBACK 8
#endif
constexpr int kLookback = DARBS_RADIX_LOOKBACK;  // predecessors read per round trip

struct Plan {  // the digits of one sort, least significant first
    int passes;
    int shift[kMaxPasses];
    int bits[kMaxPasses];
};

__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(unsigned* p, unsigned v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Exclusive scan of one value per thread over the first kBins threads of the CTA (threads beyond
// them pass 0 and take part in the barriers).  `ws` holds kBins / 32 words.
__device__ __forceinline__ unsigned scan_bins(unsigned v, unsigned* ws) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (warp < kBins / 32 && lane == 31) ws[warp] = inc;
    __syncthreads();
    unsigned base = 0;
    if (warp < kBins / 32)
        for (int w = 0; w < warp; ++w) base += ws[w];
    __syncthreads();
    return base + inc - v;
}

// The same for two values at once (one pair of barriers).
__device__ __forceinline__ uint2 scan_bins2(unsigned a, unsigned b, uint2* ws) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned ia = a, ib = b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned ta = __shfl_up_sync(0xffffffffu, ia, o), tb = __shfl_up_sync(0xffffffffu, ib, o);
        if (lane >= o) {
            ia += ta;
            ib += tb;
        }
    }
    if (warp < kBins / 32 && lane == 31) ws[warp] = make_uint2(ia, ib);
    __syncthreads();
    unsigned ba = 0, bb = 0;
    if (warp < kBins / 32)
        for (int w = 0; w < warp; ++w) {
            const uint2 t = ws[w];
            ba += t.x;
            bb += t.y;
        }
    return make_uint2(ba + ia - a, bb + ib - b);
}

// ---------------------------------------------------------------- digit histograms of all passes
template <typename KeyT, int THREADS>
__device__ __forceinline__ void histogram_body(const KeyT* __restrict__ keys, unsigned n, const Plan& plan,
                                               unsigned* __restrict__ hist) {
    __shared__ unsigned sh[kMaxPasses * kBins];
    for (int i = threadIdx.x; i < kMaxPasses * kBins; i += THREADS) sh[i] = 0;
    __syncthreads();
    constexpr int kVec = 16 / sizeof(KeyT);
    auto count = [&](unsigned k) {
#pragma unroll
        for (int p = 0; p < kMaxPasses; ++p)
            if (p < plan.passes) atomicAdd(&sh[p * kBins + ((k >> plan.shift[p]) & ((1u << plan.bits[p]) - 1u))], 1u);
    };
    const unsigned nvec = ((reinterpret_cast<uintptr_t>(keys) & 15) == 0) ? n / kVec : 0;
    for (unsigned i = blockIdx.x * THREADS + threadIdx.x; i < nvec; i += gridDim.x * THREADS) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(keys) + i);
        const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if constexpr (sizeof(KeyT) == 4) {
                count(w[j]);
            } else {
                count(w[j] & 0xffffu);
                count(w[j] >> 16);
            }
        }
    }
    for (unsigned i = nvec * kVec + blockIdx.x * THREADS + threadIdx.x; i < n; i += gridDim.x * THREADS)
        count((unsigned)keys[i]);
    __syncthreads();
    for (int i = threadIdx.x; i < plan.passes * kBins; i += THREADS)
        if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

template <typename KeyT, int THREADS>
__global__ void __launch_bounds__(THREADS)
histogram_kernel(const KeyT* __restrict__ keys, unsigned n, Plan plan, unsigned* __restrict__ hist) {
    histogram_body<KeyT, THREADS>(keys, n, plan, hist);
}

constexpr int kHistogramThreads = 512;
inline unsigned histogram_blocks(unsigned n, int sms) {
    unsigned blocks = (n + kHistogramThreads * 16 - 1) / (kHistogramThreads * 16);
    return blocks > (unsigned)(4 * sms) ? (unsigned)(4 * sms) : blocks;
}

// ---------------------------------------------------------------- one pass
template <typename KeyT, int THREADS, int ITEMS>
struct PassShape {
    static constexpr int kWarps = THREADS / 32;
    static constexpr int kChunk = THREADS * ITEMS;
    // warp counters + warp peer tables + the reorder buffers
    static constexpr size_t kSmem = sizeof(unsigned) * 2 * kWarps * kBins + (sizeof(unsigned) + sizeof(KeyT)) * kChunk;
};

#ifdef DARBS_RADIX_PROFILE
#define RADIX_MARK() do { t_[tn_++] = clock64(); } while (0)
#else
#define RADIX_MARK() do {} while (0)
#endif

// FULL: every slot of the chunk holds a key of the input (all chunks but the last).
template <typename KeyT, int THREADS, int ITEMS, bool FULL>
__device__ __forceinline__ void pass_body(const KeyT* __restrict__ keys_in, const unsigned* __restrict__ vals_in,
                                          KeyT* __restrict__ keys_out, unsigned* __restrict__ vals_out, unsigned n,
                                          int shift, unsigned mask, const unsigned* __restrict__ ghist,
                                          unsigned* __restrict__ status, unsigned chunk, unsigned* warp_hist,
                                          unsigned* warp_peer, unsigned* s_vals, KeyT* s_keys, unsigned* s_base,
                                          unsigned* s_start, uint2* s_ws
#ifdef DARBS_RADIX_PROFILE
                                          , long long* t_, int& tn_
#endif
) {
    using Shape = PassShape<KeyT, THREADS, ITEMS>;
    constexpr int kWarps = Shape::kWarps, kChunk = Shape::kChunk;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned first = chunk * (unsigned)kChunk;

    // keys, warp-striped: item i of lane l of warp w is element w * 32 * ITEMS + i * 32 + l
    const unsigned wbase = first + (unsigned)(warp * 32 * ITEMS + lane);
    const KeyT* kin = keys_in + wbase;
    const unsigned n_items = FULL ? (unsigned)ITEMS : (wbase < n ? (n - wbase + 31) / 32 : 0u);  // of this lane
    KeyT key[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) key[i] = (FULL || (unsigned)i < n_items) ? kin[i * 32] : (KeyT)0;
    const unsigned gcount = tid < kBins ? ghist[tid] : 0u;
    RADIX_MARK();

    // Rank within (warp, digit).  The lanes of a step that hold an equal digit find each other
    // through the warp's peer table in shared memory: every lane ORs its bit into the digit's
    // word, reads the word back, and the group's highest lane advances the warp's private counter
    // and clears the word.  Measured on B200 per 32 keys: 7 SM-cycles for random digits, 34 when
    // all are equal; eight ballots (VOTE issues once per 8 cycles) cost 25; match.any is microcoded,
    // ~45 cycles per distinct value, 1400 for random digits.
    unsigned* wh = warp_hist + warp * kBins;
    unsigned* wp = warp_peer + warp * kBins;
    const unsigned lt = (1u << lane) - 1u, me = 1u << lane;
    static_assert(ITEMS % 2 == 0 && THREADS * ITEMS <= 65536, "ranks are packed two to a register");
    unsigned rank2[ITEMS / 2];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const bool valid = FULL || (unsigned)i < n_items;
        const unsigned d = ((unsigned)key[i] >> shift) & mask;
        if (valid) atomicOr(&wp[d], me);
        __syncwarp();
        unsigned m = me, old = 0;
        if (valid) {
            m = wp[d];
            old = wh[d];
        }
        __syncwarp();
        const unsigned r = __popc(m & lt);
        if (valid && (m >> lane) == 1u) {  // the group's highest lane: r + 1 members
            wh[d] = old + r + 1u;
            wp[d] = 0u;
        }
        __syncwarp();
        const unsigned rr = old + r;  // < 2^16
        rank2[i >> 1] = (i & 1) ? (rank2[i >> 1] | (rr << 16)) : rr;
    }
    __syncthreads();
    RADIX_MARK();

    // per digit: exclusive prefix over the warps, the chunk's count -> published at once
    unsigned count = 0;
    if (tid < kBins) {
#pragma unroll 4
        for (int w = 0; w < kWarps; ++w) {
            const unsigned t = warp_hist[w * kBins + tid];
            warp_hist[w * kBins + tid] = count;
            count += t;
        }
        st_relaxed(status + (size_t)chunk * kBins + tid, count | (chunk == 0 ? kInclusive : kPartial));
    }
    const uint2 starts = scan_bins2(count, gcount, s_ws);
    const unsigned local_start = starts.x, global_start = starts.y;
    if (tid < kBins) s_start[tid] = local_start;
    __syncthreads();
    RADIX_MARK();

    // reorder into shared memory (the values are loaded only now: 16 more live registers during the
    // rank loop would spill at two CTAs of 512 threads per SM — measured, no faster)
    const unsigned* vin = vals_in + wbase;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        if (FULL || (unsigned)i < n_items) {
            const unsigned d = ((unsigned)key[i] >> shift) & mask;
            const unsigned pos = s_start[d] + wh[d] + ((rank2[i >> 1] >> (16 * (i & 1))) & 0xffffu);
            s_keys[pos] = key[i];
            s_vals[pos] = vin[i * 32];
        }
    }
    RADIX_MARK();

    // decoupled look-back: equal-digit keys in all earlier chunks
    if (tid < kBins) {
        unsigned excl = 0;
        if (chunk > 0) {
            long long c = (long long)chunk - 1;
            bool done = false;
            while (!done) {
                unsigned s[kLookback];
#pragma unroll
                for (int j = 0; j < kLookback; ++j)
                    s[j] = c - j >= 0 ? ld_relaxed(status + (size_t)(c - j) * kBins + tid) : kInclusive;
                int j = 0;
#pragma unroll
                for (; j < kLookback; ++j) {
                    const unsigned flag = s[j] >> 30;
                    if (flag == 0) break;  // not published yet: poll again from here
                    excl += s[j] & kValue;
                    if (flag == 2) {
                        done = true;
                        break;
                    }
                }
                c -= j;
            }
            st_relaxed(status + (size_t)chunk * kBins + tid, (excl + count) | kInclusive);
        }
        s_base[tid] = global_start + excl - local_start;
    }
    __syncthreads();
    RADIX_MARK();

    // every digit's keys leave as one contiguous run
    const unsigned valid_count = FULL ? (unsigned)kChunk : n - first;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const unsigned j = (unsigned)(i * THREADS + tid);
        if (FULL || j < valid_count) {
            const KeyT k = s_keys[j];
            const unsigned pos = s_base[((unsigned)k >> shift) & mask] + j;
            keys_out[pos] = k;
            vals_out[pos] = s_vals[j];
        }
    }
    RADIX_MARK();
}

// keys_in/vals_in -> keys_out/vals_out, stable by digit (key >> shift) & (2^bits - 1).
// ghist: this digit's histogram over the whole input.  status: [chunks][kBins], zeroed.  ticket: zeroed.
template <typename KeyT, int THREADS, int ITEMS>
__global__ void __launch_bounds__(THREADS, 1024 / THREADS)
onesweep_kernel(const KeyT* __restrict__ keys_in, const unsigned* __restrict__ vals_in,
                KeyT* __restrict__ keys_out, unsigned* __restrict__ vals_out, unsigned n_bound,
                const unsigned long long* __restrict__ n_dev, int shift, int bits,
                const unsigned* __restrict__ ghist, unsigned* __restrict__ status, unsigned* __restrict__ ticket
#ifdef DARBS_RADIX_PROFILE
                , long long* __restrict__ prof
#endif
) {
    using Shape = PassShape<KeyT, THREADS, ITEMS>;
    constexpr int kWarps = Shape::kWarps, kChunk = Shape::kChunk;
    static_assert(THREADS >= kBins, "one thread per bin");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned* warp_hist = reinterpret_cast<unsigned*>(smem_raw);   // [kWarps][kBins]
    unsigned* warp_peer = warp_hist + kWarps * kBins;              // [kWarps][kBins]
    unsigned* s_vals = warp_peer + kWarps * kBins;                 // [kChunk]
    KeyT* s_keys = reinterpret_cast<KeyT*>(s_vals + kChunk);       // [kChunk]
    __shared__ unsigned s_base[kBins];   // output position of local slot j of a bin = s_base[bin] + j
    __shared__ unsigned s_start[kBins];  // first local slot of the bin
    __shared__ uint2 s_ws[kBins / 32];
    __shared__ unsigned s_chunk;
#ifdef DARBS_RADIX_PROFILE
    long long t_[8];
    int tn_ = 0;
#endif
    RADIX_MARK();
    const int tid = threadIdx.x;
    if (tid == 0) s_chunk = atomicAdd(ticket, 1u);
    for (int i = tid; i < 2 * kWarps * kBins; i += THREADS) warp_hist[i] = 0;
    __syncthreads();
    const unsigned chunk = s_chunk;
    const unsigned mask = (1u << bits) - 1u;
    // the element count: the launch's bound, or (n_dev given) the count a kernel left on the device,
    // clamped to the bound the buffers were sized for; chunks past it have nothing to do
    unsigned n = n_bound;
    if (n_dev) {
        // more elements than the bound: the digit histograms count all of them, so positions would
        // leave the buffers; the producer has flagged the overflow and the sort is skipped
        const unsigned long long nd = *n_dev;
        if (nd > (unsigned long long)n_bound) return;
        n = (unsigned)nd;
    }
    if ((unsigned long long)chunk * kChunk >= n) return;
#ifdef DARBS_RADIX_PROFILE
#define RADIX_PROF_ARGS , t_, tn_
#else
#define RADIX_PROF_ARGS
#endif
    if ((chunk + 1u) * (unsigned)kChunk <= n)
        pass_body<KeyT, THREADS, ITEMS, true>(keys_in, vals_in, keys_out, vals_out, n, shift, mask, ghist, status, chunk,
                                              warp_hist, warp_peer, s_vals, s_keys, s_base, s_start, s_ws RADIX_PROF_ARGS);
    else
        pass_body<KeyT, THREADS, ITEMS, false>(keys_in, vals_in, keys_out, vals_out, n, shift, mask, ghist, status, chunk,
                                               warp_hist, warp_peer, s_vals, s_keys, s_base, s_start, s_ws RADIX_PROF_ARGS);
#undef RADIX_PROF_ARGS
#ifdef DARBS_RADIX_PROFILE
    if (tid == 0 && (chunk == 0 || chunk == gridDim.x - 1)) {
        long long* o = prof + (chunk == 0 ? 0 : 8);
        for (int i = 0; i < tn_; ++i) o[i] = t_[i] - t_[0];
    }
#endif
}
#undef RADIX_MARK

// ---------------------------------------------------------------- host side
// Workspace of one sort, in 32-bit words: kTicketWords tickets (one per pass), kHistWords of digit
// histograms [pass][kBins], then the status words [pass][chunk][kBins].
constexpr size_t kTicketWords = 16, kHistWords = (size_t)kMaxPasses * kBins;
constexpr size_t kHistAt = kTicketWords, kStatusAt = kHistAt + kHistWords;
#ifndef DARBS_RADIX_THREADS
#define DARBS_RADIX_THREADS 512
#define DARBS_RADIX_ITEMS 16
#endif
constexpr int kPassThreads = DARBS_RADIX_THREADS, kPassItems = DARBS_RADIX_ITEMS;
constexpr unsigned kPassChunk = kPassThreads * kPassItems;

inline size_t chunks_of(size_t n) { return (n + kPassChunk - 1) / kPassChunk; }
inline size_t workspace_words(size_t n, int passes) { return kStatusAt + (size_t)passes * chunks_of(n) * kBins; }

template <typename KeyT>
inline cudaError_t launch_histogram(const KeyT* keys, unsigned n, const Plan& plan, unsigned* hist, int sms,
                                    cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    histogram_kernel<KeyT, kHistogramThreads><<<histogram_blocks(n, sms), kHistogramThreads, 0, stream>>>(keys, n, plan, hist);
    return cudaGetLastError();
}

#ifdef DARBS_RADIX_PROFILE
static long long* g_prof = nullptr;
#endif
// All passes of `plan` over n pairs, ping-ponging between (k0, v0) and (k1, v1).  hist: the
// digit histograms [pass][kBins], complete; tickets[pass] and status[pass][chunk][kBins] zero.
// n_dev (optional): the true count lives on the device and n is only its bound (buffers, grid).
// The sorted pairs end in buffer (plan.passes & 1).
template <typename KeyT>
inline cudaError_t launch_passes(KeyT* k0, unsigned* v0, KeyT* k1, unsigned* v1, unsigned n, const Plan& plan,
                                 unsigned* tickets, const unsigned* hist, unsigned* status, cudaStream_t stream,
                                 const unsigned long long* n_dev = nullptr) {
    if (n == 0) return cudaSuccess;
    using Shape = PassShape<KeyT, kPassThreads, kPassItems>;
    auto kernel = onesweep_kernel<KeyT, kPassThreads, kPassItems>;
    static bool configured = false;  // per KeyT instantiation
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Shape::kSmem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    const unsigned chunks = (unsigned)chunks_of(n);
    for (int p = 0; p < plan.passes; ++p) {
        const bool fwd = (p & 1) == 0;
        kernel<<<chunks, kPassThreads, Shape::kSmem, stream>>>(
            fwd ? k0 : k1, fwd ? v0 : v1, fwd ? k1 : k0, fwd ? v1 : v0, n, n_dev, plan.shift[p], plan.bits[p],
            hist + (size_t)p * kBins, status + (size_t)p * chunks * kBins, tickets + p
#ifdef DARBS_RADIX_PROFILE
            , g_prof
#endif
        );
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace radix
}  // namespace darbs_b200
