// binning.cu — device restatement of darbs::bin_splats (reference
// src/rasterizer.cpp:25-53): global stable depth order, per-splat inclusive tile
// rectangle, per-tile depth-ordered index lists.  Every kernel on the path is written here or in
// radix.cuh; no library sort or scan is called.
//
// Two-level sort instead of one wide (tile, depth) key:
//   1. stable LSD radix sort of the N (depth bits, index) pairs  -> depth order
//      (stability gives the reference's index tie-break, rasterizer.cpp:33): digit histograms of
//      the keys, then four 8-bit passes of radix.cuh;
//   2. expand_kernel, one pass IN DEPTH ORDER: the tiles-touched counts are scanned (chained
//      through decoupled look-back over the CTAs), every splat emits its (tile, index) pairs at
//      its offset — the K entries are therefore depth-ordered globally, a warp writes the entries
//      of its 32 splats as one contiguous run — and the digit histograms of the tile sort are
//      accumulated on the way, per SPLAT (a rectangle of nx x ny tiles adds ny to nx column
//      digits and nx to ny row digits: ~4 shared-memory atomics per splat, not 2 per entry);
//   3. stable radix sort of the K entries on the tile only: the key is (tile row, tile column)
//      packed, 8 + 8 bits while both fit (16 + 16 otherwise), so one pass per coordinate byte
//      (two at every size of BASELINE.json) keeps depth order inside a tile;
//   4. tile ranges from the sorted keys.
// The tile rectangle is evaluated in FP64 on the float32 inputs so that
// floor((mu -+ R)/16) is decided on exactly the values the FP64 reference sees
// (rasterizer.cpp:40-45).
#include "radix.cuh"
#include "splat.cuh"

namespace darbs_b200 {

namespace {

struct Scalars {  // lives behind the 8 work counters in ctx->counters
    unsigned long long total_entries;
    unsigned long long skipped_nonfinite;
};

__global__ void rect_kernel(int64_t n, const float* __restrict__ mu2,
                            const float* __restrict__ conic, const float* __restrict__ radius,
                            const float* __restrict__ depth, const int* __restrict__ valid,
                            int tiles_x, int tiles_y, uint2* __restrict__ rects,
                            unsigned* __restrict__ touched, unsigned* __restrict__ depth_keys,
                            unsigned* __restrict__ order, Scalars* __restrict__ scalars,
                            unsigned long long* __restrict__ k_slots) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    depth_keys[i] = depth_to_key(depth[i]);
    order[i] = (unsigned)i;
    uint2 rect;
    unsigned cnt;
    splat_rect(valid ? valid[i] != 0 : true, mu2[2 * i], mu2[2 * i + 1], conic[3 * i], conic[3 * i + 1],
               conic[3 * i + 2], radius[i], tiles_x, tiles_y, &scalars->skipped_nonfinite, rect, cnt);
    rects[i] = rect;
    touched[i] = cnt;
    accumulate_tile_count(cnt, k_slots);
}

// K, the total of the per-splat tile counts (accumulated over kSlotsK addresses by the kernel
// that made the rectangles), goes to the device scalars and straight into pinned host memory
// (mapped under UVA): the host needs it to size the tile sort, and a write from the SM does not
// queue behind a bulk host <-> device copy that may be in flight on the copy engines.  It is
// known before the depth sort starts, so the host reads it while the GPU sorts.  The kernel that
// counts the depth keys' digit histograms (the first of the sort) does it on the side.
__global__ void __launch_bounds__(radix::kHistogramThreads)
depth_histogram_kernel(const unsigned* __restrict__ keys, unsigned n, radix::Plan plan, unsigned* __restrict__ hist,
                       const unsigned long long* __restrict__ k_slots, Scalars* __restrict__ scalars,
                       volatile unsigned long long* host_total) {
    if (blockIdx.x == 0 && threadIdx.x < 32) {
        unsigned long long k = k_slots[threadIdx.x] + k_slots[threadIdx.x + 32];
        for (int o = 16; o > 0; o >>= 1) k += __shfl_xor_sync(0xffffffffu, k, o);
        if (threadIdx.x == 0) {
            scalars->total_entries = k;
            *host_total = k;
            __threadfence_system();
        }
    }
    radix::histogram_body<unsigned, radix::kHistogramThreads>(keys, n, plan, hist);
}
static_assert(kSlotsK == 64, "total_kernel sums two slots per lane");

// TileKey: (tile row << 8 | tile column) in an unsigned short while both coordinates fit a byte
// (every size of BASELINE.json: 120 x 68 tiles at 1080p, 240 x 135 at 4K), (row << 16 | column) in
// an unsigned otherwise.  A tile-sort pass then moves 6 bytes per entry, not 8.
template <typename TileKey>
struct TilePack {
    static constexpr int kRowShift = sizeof(TileKey) == 2 ? 8 : 16;
    static constexpr unsigned kColMask = (1u << kRowShift) - 1u;
    __host__ __device__ static TileKey pack(unsigned tx, unsigned ty) { return (TileKey)((ty << kRowShift) | tx); }
    __host__ __device__ static unsigned tile_of(TileKey k, int tiles_x) {
        return ((unsigned)k >> kRowShift) * (unsigned)tiles_x + ((unsigned)k & kColMask);
    }
};

constexpr int kExpandThreads = 256, kExpandItems = 8;
constexpr int kExpandChunk = kExpandThreads * kExpandItems;  // depth ranks per CTA

// Step 2 of the header.  status[chunks] and ticket zeroed; hist = the tile sort's digit histograms
// [pass][256], zeroed.  plan.passes may be 0 (a single tile).
template <typename TileKey, bool BYTE_DIGITS>
__global__ void __launch_bounds__(kExpandThreads)
expand_kernel(unsigned n, const unsigned* __restrict__ order, const uint2* __restrict__ rects,
              const unsigned* __restrict__ touched, radix::Plan plan, unsigned* __restrict__ hist,
              unsigned* __restrict__ status, unsigned* __restrict__ ticket, TileKey* __restrict__ tile_keys,
              unsigned* __restrict__ tile_vals, unsigned capacity, unsigned long long* __restrict__ overflow) {
    using Pack = TilePack<TileKey>;
    __shared__ unsigned s_hist[radix::kMaxPasses * radix::kBins];
    __shared__ unsigned s_wtot[kExpandThreads / 32];
    __shared__ unsigned s_chunk, s_base;
    const unsigned full = 0xffffffffu;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_chunk = atomicAdd(ticket, 1u);
    for (int i = tid; i < plan.passes * radix::kBins; i += kExpandThreads) s_hist[i] = 0;
    __syncthreads();
    const unsigned chunk = s_chunk;
    const unsigned first = chunk * (unsigned)kExpandChunk + (unsigned)(warp * kExpandItems * 32 + lane);

    // this lane's splats: ranks first + 32 i
    unsigned idx[kExpandItems], cnt[kExpandItems];
    uint2 rect[kExpandItems];
#pragma unroll
    for (int i = 0; i < kExpandItems; ++i) {
        const unsigned r = first + 32u * i;
        idx[i] = r < n ? order[r] : 0u;
    }
#pragma unroll
    for (int i = 0; i < kExpandItems; ++i) {
        const bool ok = first + 32u * i < n;
        cnt[i] = ok ? touched[idx[i]] : 0u;
        rect[i] = ok ? rects[idx[i]] : make_uint2(0, 0);
    }
    // scan of the counts in rank order: lanes of an item, items of a warp, warps of the CTA
    unsigned rel[kExpandItems], item_total[kExpandItems], warp_total = 0;
#pragma unroll
    for (int i = 0; i < kExpandItems; ++i) {
        unsigned inc = cnt[i];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(full, inc, o);
            if (lane >= o) inc += t;
        }
        rel[i] = inc - cnt[i];
        item_total[i] = __shfl_sync(full, inc, 31);
        warp_total += item_total[i];
    }
    if (lane == 0) s_wtot[warp] = warp_total;
    __syncthreads();
    unsigned warp_base = 0, cta_total = 0;
#pragma unroll
    for (int w = 0; w < kExpandThreads / 32; ++w) {
        const unsigned t = s_wtot[w];
        if (w < warp) warp_base += t;
        cta_total += t;
    }
    if (tid == 0) radix::st_relaxed(status + chunk, cta_total | (chunk == 0 ? radix::kInclusive : radix::kPartial));
    // the tile sort's digit histograms, per splat: nx column digits get ny, ny row digits get nx
    // (after the publish: this work runs under the look-back of the CTAs behind this one)
    if (BYTE_DIGITS) {  // pass 0 = the column, pass 1 = the row: no shifts, no masks
#pragma unroll
        for (int i = 0; i < kExpandItems; ++i) {
            if (cnt[i] == 0) continue;
            const unsigned x0 = rect[i].x & 0xffffu, y0 = rect[i].x >> 16, x1 = rect[i].y & 0xffffu, y1 = rect[i].y >> 16;
            const unsigned nx = x1 - x0 + 1u, ny = y1 - y0 + 1u;
            for (unsigned x = x0; x <= x1; ++x) atomicAdd(&s_hist[x], ny);
            for (unsigned y = y0; y <= y1; ++y) atomicAdd(&s_hist[radix::kBins + y], nx);
        }
    } else {
#pragma unroll
        for (int i = 0; i < kExpandItems; ++i) {
            if (cnt[i] == 0) continue;
            const unsigned x0 = rect[i].x & 0xffffu, y0 = rect[i].x >> 16, x1 = rect[i].y & 0xffffu, y1 = rect[i].y >> 16;
            const unsigned nx = x1 - x0 + 1u, ny = y1 - y0 + 1u;
            for (int p = 0; p < plan.passes; ++p) {
                const unsigned mask = (1u << plan.bits[p]) - 1u;
                unsigned* h = s_hist + p * radix::kBins;
                if (plan.shift[p] < Pack::kRowShift) {
                    for (unsigned x = x0; x <= x1; ++x) atomicAdd(&h[(x >> plan.shift[p]) & mask], ny);
                } else {
                    const int sh = plan.shift[p] - Pack::kRowShift;
                    for (unsigned y = y0; y <= y1; ++y) atomicAdd(&h[(y >> sh) & mask], nx);
                }
            }
        }
    }
    // entries of all earlier CTAs: decoupled look-back, 128 predecessors per round trip (every CTA
    // of a million-splat view is resident at once, so the walk is rounds of L2 latency, not waiting)
    if (warp == 0) {
        unsigned excl = 0;
        long long c = (long long)chunk - 1;
        while (c >= 0) {
            constexpr int kRounds = 4;
            unsigned s[kRounds];
#pragma unroll
            for (int r = 0; r < kRounds; ++r) {
                const long long at = c - 32 * r - lane;
                s[r] = at >= 0 ? radix::ld_relaxed(status + at) : radix::kInclusive;
            }
            bool done = false;
            int used = 0;
#pragma unroll
            for (int r = 0; r < kRounds; ++r) {
                if (done) continue;
                if (!__all_sync(full, (s[r] >> 30) != 0u)) {  // someone has not published yet: poll again from here
                    done = true;
                    continue;
                }
                const unsigned incl = __ballot_sync(full, (s[r] >> 30) == 2u);
                const int stop = incl ? __ffs(incl) - 1 : 31;
                unsigned v = lane <= stop ? (s[r] & radix::kValue) : 0u;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(full, v, o);
                excl += v;
                used = r + 1;
                if (incl) {
                    done = true;
                    c = -1 - 32 * used;  // leaves the walk
                }
            }
            c -= 32 * used;
        }
        if (lane == 0) {
            if (chunk > 0) radix::st_relaxed(status + chunk, (excl + cta_total) | radix::kInclusive);
            s_base = excl;
        }
    }
    __syncthreads();
    unsigned base = s_base + warp_base;

    // A warp writes the entries of 32 consecutive ranks TOGETHER: entry e of the run is written by
    // lane e mod 32, which finds the owning splat by a binary search over the lanes' offsets, so
    // the writes are one contiguous run instead of 32 interleaved short ones (rasterizer.cpp:46-50).
#pragma unroll
    for (int i = 0; i < kExpandItems; ++i) {
        const unsigned total = item_total[i];
        // lanes past n hold count 0: their offset equals the end of the run and is never chosen
        for (unsigned e0 = 0; e0 < total; e0 += 32) {  // warp-uniform trip count: the shuffles need every lane
            const unsigned e = e0 + lane;
            int lo = 0;  // largest lane whose offset is <= e (zero-count lanes share the offset of the next)
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const unsigned probe = __shfl_sync(full, rel[i], min(lo + step, 31));
                if (lo + step <= 31 && probe <= e) lo += step;
            }
            const unsigned o_rel = __shfl_sync(full, rel[i], lo);
            const unsigned o_idx = __shfl_sync(full, idx[i], lo);
            const unsigned rx = __shfl_sync(full, rect[i].x, lo), ry = __shfl_sync(full, rect[i].y, lo);
            const unsigned x0 = rx & 0xffffu, y0 = rx >> 16, w = (ry & 0xffffu) - x0 + 1u;
            if (e < total && base + e < capacity) {  // capacity: what the entry buffers were sized for
                const unsigned q = e - o_rel;
                const unsigned qy = q / w, qx = q - qy * w;
                tile_keys[base + e] = Pack::pack(x0 + qx, y0 + qy);
                tile_vals[base + e] = o_idx;
            }
        }
        base += total;
    }
    // more entries than the caller's capacity (darbs_cuda_set_entry_capacity): the view is incomplete
    if (tid == 0 && (unsigned long long)s_base + cta_total > capacity) *overflow = 1ull;
    __syncthreads();
    for (int i = tid; i < plan.passes * radix::kBins; i += kExpandThreads)
        if (s_hist[i]) atomicAdd(&hist[i], s_hist[i]);
}

template <typename TileKey>
__global__ void ranges_kernel(int64_t k_bound, const unsigned long long* __restrict__ k_dev,
                              const TileKey* __restrict__ sorted_tiles, int tiles_x, int2* __restrict__ ranges) {
    // eight consecutive entries per thread: one boundary test per entry against its predecessor
    constexpr int kPer = 8;
    int64_t k = k_bound;  // or the count on the device; beyond the bound nothing was sorted: no ranges
    if (k_dev) {
        if (*k_dev > (unsigned long long)k_bound) return;
        k = (int64_t)*k_dev;
    }
    const int64_t first = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * kPer;
    if (first >= k) return;
    unsigned prev = first > 0 ? TilePack<TileKey>::tile_of(sorted_tiles[first - 1], tiles_x) : 0xffffffffu;
    const int64_t stop = first + kPer < k ? first + kPer : k;
    for (int64_t i = first; i < stop; ++i) {
        const unsigned t = TilePack<TileKey>::tile_of(sorted_tiles[i], tiles_x);
        if (t != prev) {
            ranges[t].x = (int)i;
            if (prev != 0xffffffffu) ranges[prev].y = (int)i;
        }
        prev = t;
    }
    if (stop == k) ranges[prev].y = (int)k;
}

template <typename TileKey>
__global__ void export_keys_kernel(int64_t k, const TileKey* __restrict__ sorted_tiles, int tiles_x,
                                   const unsigned* __restrict__ point_list,
                                   const unsigned* __restrict__ rank_of,
                                   unsigned long long* __restrict__ keys) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= k) return;
    keys[i] = ((unsigned long long)TilePack<TileKey>::tile_of(sorted_tiles[i], tiles_x) << 32) | rank_of[point_list[i]];
}

__global__ void invert_order_kernel(int64_t n, const unsigned* __restrict__ order,
                                    unsigned* __restrict__ rank_of) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r < n) rank_of[order[r]] = (unsigned)r;
}

inline unsigned grid_for(int64_t n, int threads) { return (unsigned)((n + threads - 1) / threads); }

int bits_for(int tiles) {
    int b = 1;
    while ((1 << b) < tiles) ++b;
    return b;
}

// The sort workspace ctx->sort_ws, in 32-bit words.  One memset clears all of it per call:
//   depth sort:  tickets | digit histograms | status [4][chunks(n)][256]
//   expand:      ticket | status [expand chunks(n)]
//   tile sort:   tickets | digit histograms          (its status words: ctx->tile_status, sized by K)
struct SortWorkspace {
    unsigned *depth_tickets, *depth_hist, *depth_status;
    unsigned *expand_ticket, *expand_status;
    unsigned *tile_tickets, *tile_hist;
    size_t words;
};
constexpr int kDepthPasses = 4;

SortWorkspace sort_workspace(darbs_cuda_ctx* ctx, int64_t n) {
    SortWorkspace w;
    unsigned* p = (unsigned*)ctx->sort_ws.ptr;
    const size_t nn = (size_t)(n > 0 ? n : 1);
    w.depth_tickets = p;
    w.depth_hist = p + radix::kTicketWords;
    w.depth_status = w.depth_hist + radix::kHistWords;
    w.expand_ticket = w.depth_status + (size_t)kDepthPasses * radix::chunks_of(nn) * radix::kBins;
    w.expand_status = w.expand_ticket + 16;
    w.tile_tickets = w.expand_status + ((nn + kExpandChunk - 1) / kExpandChunk + 15) / 16 * 16;
    w.tile_hist = w.tile_tickets + radix::kTicketWords;
    w.words = (size_t)(w.tile_hist + radix::kHistWords - p);
    return w;
}

}  // namespace

const int32_t* point_list_ptr(const darbs_cuda_ctx* ctx) {
    return (const int32_t*)ctx->tile_vals.ptr + (size_t)ctx->cur_key_buf * (ctx->tile_vals.bytes / 8);
}
const uint32_t* depth_order_ptr(const darbs_cuda_ctx* ctx) {
    return (const uint32_t*)ctx->order.ptr + (size_t)ctx->cur_order_buf * (ctx->order.bytes / 8);
}

// The digits of the tile sort: one pass per coordinate byte that can differ, columns first.
template <typename TileKey>
radix::Plan tile_plan(int tiles_x, int tiles_y) {
    radix::Plan plan = {};
    auto add = [&](int dim, int base) {
        if (dim <= 1) return;  // a single column or row: the digit is constant
        const int bits = bits_for(dim);
        for (int lo = 0; lo < bits; lo += 8) {
            plan.shift[plan.passes] = base + lo;
            plan.bits[plan.passes] = bits - lo < 8 ? bits - lo : 8;
            ++plan.passes;
        }
    };
    add(tiles_x, 0);
    add(tiles_y, TilePack<TileKey>::kRowShift);
    return plan;
}

// The render kernels' CTAs take the tiles longest list first: a tile's work grows with its list, the
// hardware hands CTAs out in index order, and with the long ones started first the launch's tail is
// made of short ones (raster order leaves whatever the bottom rows of the image hold for last).
// One CTA: counting sort of the tiles by list length in buckets of 16 entries (order inside a
// bucket is whatever the atomics give: it only decides when a tile runs, never what it computes).
constexpr int kOrderBuckets = 512;
constexpr int kOrderThreads = 1024, kOrderRegs = 8;  // up to 8192 tiles keep their lengths in registers
__device__ __forceinline__ int order_bucket(int len) { return min(kOrderBuckets - 1, len >> 4); }
__global__ void __launch_bounds__(kOrderThreads) tile_order_kernel(const int2* __restrict__ ranges, int tiles,
                                                                   int* __restrict__ order) {
    __shared__ int cursor[kOrderBuckets];
    for (int b = threadIdx.x; b < kOrderBuckets; b += kOrderThreads) cursor[b] = 0;
    int len[kOrderRegs];
#pragma unroll
    for (int i = 0; i < kOrderRegs; ++i) {  // independent loads, all in flight at once
        const int t = threadIdx.x + i * kOrderThreads;
        len[i] = -1;
        if (t < tiles) {
            const int2 r = ranges[t];
            len[i] = r.y - r.x;
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kOrderRegs; ++i)
        if (len[i] >= 0) atomicAdd(&cursor[order_bucket(len[i])], 1);
    for (int t = threadIdx.x + kOrderRegs * kOrderThreads; t < tiles; t += kOrderThreads) {
        const int2 r = ranges[t];
        atomicAdd(&cursor[order_bucket(r.y - r.x)], 1);
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // exclusive scan from the longest bucket down: 16 buckets per lane
        constexpr int kPer = kOrderBuckets / 32;
        const int top = kOrderBuckets - 1 - (int)threadIdx.x * kPer;  // this lane's longest bucket
        int sum = 0;
        for (int i = 0; i < kPer; ++i) sum += cursor[top - i];
        int incl = sum;
        for (int d = 1; d < 32; d <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, d);
            if ((int)threadIdx.x >= d) incl += v;
        }
        int run = incl - sum;
        for (int i = 0; i < kPer; ++i) {
            const int c = cursor[top - i];
            cursor[top - i] = run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kOrderRegs; ++i)
        if (len[i] >= 0) order[atomicAdd(&cursor[order_bucket(len[i])], 1)] = threadIdx.x + i * kOrderThreads;
    for (int t = threadIdx.x + kOrderRegs * kOrderThreads; t < tiles; t += kOrderThreads) {
        const int2 r = ranges[t];
        order[atomicAdd(&cursor[order_bucket(r.y - r.x)], 1)] = t;
    }
}

// Steps 2-4 of the header.  The small part of the sort workspace (tickets, histograms, the
// expand kernel's status words) was cleared by binning_begin; the status words of the tile passes
// depend on K and are cleared here.
template <typename TileKey>
// k: the entry count, or (k_dev given) the capacity the caller vouches for while the count stays on the device.
darbs_status tile_sort(darbs_cuda_ctx* ctx, int64_t n, int64_t k, const unsigned long long* k_dev,
                       const unsigned* order, const uint2* rects, const unsigned* touched) {
    cudaStream_t s = ctx->stream;
    DARBS_TRY(reserve(ctx, ctx->tile_keys, sizeof(unsigned) * 2 * (size_t)k));  // sized for 32-bit keys
    DARBS_TRY(reserve(ctx, ctx->tile_vals, sizeof(unsigned) * 2 * (size_t)k));
    TileKey* tk0 = (TileKey*)ctx->tile_keys.ptr;
    TileKey* tk1 = (TileKey*)((unsigned*)ctx->tile_keys.ptr + ctx->tile_keys.bytes / 8);
    unsigned* tv0 = (unsigned*)ctx->tile_vals.ptr;
    unsigned* tv1 = tv0 + ctx->tile_vals.bytes / 8;
    const radix::Plan plan = tile_plan<TileKey>(ctx->tiles_x, ctx->tiles_y);
    SortWorkspace ws = sort_workspace(ctx, n);
    const size_t status_words = (size_t)plan.passes * radix::chunks_of((size_t)k) * radix::kBins;
    DARBS_TRY(reserve(ctx, ctx->tile_status, sizeof(unsigned) * (status_words ? status_words : 1)));
    if (status_words)
        DARBS_CUDA_TRY(ctx, cudaMemsetAsync(ctx->tile_status.ptr, 0, sizeof(unsigned) * status_words, s));

    // pass 0 = the column byte, pass 1 = the row byte: the histograms need neither shifts nor masks
    const bool byte_digits = sizeof(TileKey) == 2 && plan.passes == 2 && plan.shift[1] == 8;
    unsigned long long* overflow = (unsigned long long*)ctx->counters.ptr + kOverflowAt;
    if (byte_digits)
        expand_kernel<TileKey, true><<<grid_for(n, kExpandChunk), kExpandThreads, 0, s>>>(
            (unsigned)n, order, rects, touched, plan, ws.tile_hist, ws.expand_status, ws.expand_ticket, tk0, tv0,
            (unsigned)k, overflow);
    else
        expand_kernel<TileKey, false><<<grid_for(n, kExpandChunk), kExpandThreads, 0, s>>>(
            (unsigned)n, order, rects, touched, plan, ws.tile_hist, ws.expand_status, ws.expand_ticket, tk0, tv0,
            (unsigned)k, overflow);
    DARBS_TRY(check_launch(ctx, "expand_kernel"));
    DARBS_CUDA_TRY(ctx, radix::launch_passes<TileKey>(tk0, tv0, tk1, tv1, (unsigned)k, plan, ws.tile_tickets,
                                                      ws.tile_hist, (unsigned*)ctx->tile_status.ptr, s, k_dev));
    ctx->launches += plan.passes;
    ctx->cur_key_buf = plan.passes & 1;
    const TileKey* sorted_tiles = ctx->cur_key_buf ? tk1 : tk0;
    ranges_kernel<TileKey><<<grid_for(((int64_t)k + 7) / 8, 256), 256, 0, s>>>((int64_t)k, k_dev, sorted_tiles,
                                                                              ctx->tiles_x, (int2*)ctx->ranges.ptr);
    DARBS_TRY(check_launch(ctx, "ranges_kernel"));
    if (ctx->tile_order_wanted) {
        // on a second stream, under the cull kernel (which takes the tiles in raster order: neighbours
        // share records); the forward's launch waits for it (render.cu join_tile_order)
        const int tiles = ctx->tiles_x * ctx->tiles_y;
        DARBS_CUDA_TRY(ctx, cudaEventRecord(ctx->ranges_ready, s));
        DARBS_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->aux_stream, ctx->ranges_ready, 0));
        tile_order_kernel<<<1, kOrderThreads, 0, ctx->aux_stream>>>((const int2*)ctx->ranges.ptr, tiles,
                                                                   (int*)ctx->tile_order.ptr);
        DARBS_TRY(check_launch(ctx, "tile_order_kernel"));
        DARBS_CUDA_TRY(ctx, cudaEventRecord(ctx->order_ready, ctx->aux_stream));
        ctx->tile_order_valid = true;
        ctx->tile_order_pending = true;
    }
    return DARBS_OK;
}

// Sizes the per-splat buffers of the stage, clears its counters and the tile ranges, and tells
// where a fused preprocess may leave the rectangles, depth keys and identity order itself.
darbs_status binning_begin(darbs_cuda_ctx* ctx, int64_t n, int width, int height, SplatSinks* sinks) {
    cudaStream_t s = ctx->stream;
    ctx->tiles_x = (width + DARBS_TILE_SIZE - 1) / DARBS_TILE_SIZE;
    ctx->tiles_y = (height + DARBS_TILE_SIZE - 1) / DARBS_TILE_SIZE;
    const int tiles = ctx->tiles_x * ctx->tiles_y;
    if (ctx->tiles_x > 65535 || ctx->tiles_y > 65535)
        return fail(ctx, DARBS_INVALID_PARAMETER, "image too large for 16-bit tile coordinates");
    // the sort's look-back words carry 30-bit counts (radix.cuh)
    if (n >= (int64_t)1 << 30) return fail(ctx, DARBS_INVALID_PARAMETER, "too many splats (2^30 or more)");

    DARBS_TRY(reserve(ctx, ctx->ranges, sizeof(int2) * (size_t)(tiles > 0 ? tiles : 1)));
    DARBS_TRY(reserve(ctx, ctx->tile_order, sizeof(int) * (size_t)(tiles > 0 ? tiles : 1)));
    ctx->tile_order_valid = false;  // until this view's tile sort has ordered its tiles
    DARBS_CUDA_TRY(ctx, cudaMemsetAsync(ctx->ranges.ptr, 0, sizeof(int2) * (size_t)tiles, s));
    Scalars* scalars = (Scalars*)((unsigned long long*)ctx->counters.ptr + 8);
    // work counters, scalars and the K slots in one clear (what lies between them is scratch)
    unsigned long long* k_slots = (unsigned long long*)ctx->counters.ptr + kSlotsKBase;
    DARBS_CUDA_TRY(ctx, cudaMemsetAsync(ctx->counters.ptr, 0, sizeof(unsigned long long) * (kSlotsKBase + kSlotsK), s));
    ctx->fwd_entries = 0;
    ctx->cur_key_buf = 0;
    ctx->cur_order_buf = 0;
    if (sinks) *sinks = SplatSinks();
    if (n == 0 || tiles == 0) return DARBS_OK;

    const size_t nn = (size_t)n;
    DARBS_TRY(reserve(ctx, ctx->rects, sizeof(uint2) * nn + sizeof(unsigned) * nn));
    DARBS_TRY(reserve(ctx, ctx->depth_keys, sizeof(unsigned) * 2 * nn));
    DARBS_TRY(reserve(ctx, ctx->order, sizeof(unsigned) * 2 * nn));
    {
        const size_t words = sort_workspace(ctx, n).words;
        DARBS_TRY(reserve(ctx, ctx->sort_ws, sizeof(unsigned) * words));
        DARBS_CUDA_TRY(ctx, cudaMemsetAsync(ctx->sort_ws.ptr, 0, sizeof(unsigned) * words, s));
    }
    if (sinks) {
        sinks->rects = (uint2*)ctx->rects.ptr;
        sinks->touched = (unsigned*)(sinks->rects + nn);
        sinks->depth_keys = (unsigned*)ctx->depth_keys.ptr;
        sinks->order = (unsigned*)ctx->order.ptr;
        sinks->skipped_nonfinite = &scalars->skipped_nonfinite;
        sinks->k_slots = k_slots;
        sinks->tiles_x = ctx->tiles_x;
        sinks->tiles_y = ctx->tiles_y;
    }
    return DARBS_OK;
}

// rects_done: a fused preprocess already filled the sinks of binning_begin (which the caller ran).
darbs_status run_binning(darbs_cuda_ctx* ctx, int64_t n, const float* mu2, const float* conic,
                         const float* radius, const float* depth, const int32_t* valid,
                         int width, int height, bool rects_done) {
    cudaStream_t s = ctx->stream;
    if (!rects_done) DARBS_TRY(binning_begin(ctx, n, width, height, nullptr));
    const int tiles = ctx->tiles_x * ctx->tiles_y;
    if (n == 0 || tiles == 0) return DARBS_OK;
    Scalars* scalars = (Scalars*)((unsigned long long*)ctx->counters.ptr + 8);
    const size_t nn = (size_t)n;
    uint2* rects = (uint2*)ctx->rects.ptr;
    unsigned* touched = (unsigned*)(rects + nn);
    // double buffers are split at half of the RESERVED size so that the halves
    // stay put when the buffer is larger than this call needs.
    unsigned* dk0 = (unsigned*)ctx->depth_keys.ptr;
    unsigned* dk1 = dk0 + ctx->depth_keys.bytes / 8;
    unsigned* or0 = (unsigned*)ctx->order.ptr;
    unsigned* or1 = or0 + ctx->order.bytes / 8;

    if (!rects_done) {
        rect_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, mu2, conic, radius, depth, valid, ctx->tiles_x,
                                                     ctx->tiles_y, rects, touched, dk0, or0, scalars,
                                                     (unsigned long long*)ctx->counters.ptr + kSlotsKBase);
        DARBS_TRY(check_launch(ctx, "rect_kernel"));
    }
    // 1. stable depth sort: digit histograms of the keys, then four 8-bit passes.  K is complete:
    // the histogram kernel publishes it, and the host picks it up while the depth sort runs
    DARBS_TRY(reserve_pinned(ctx, 64));
    const SortWorkspace ws = sort_workspace(ctx, n);
    const radix::Plan depth_plan = {kDepthPasses, {0, 8, 16, 24}, {8, 8, 8, 8}};
    depth_histogram_kernel<<<radix::histogram_blocks((unsigned)n, ctx->sm_count), radix::kHistogramThreads, 0, s>>>(
        dk0, (unsigned)n, depth_plan, ws.depth_hist, (const unsigned long long*)ctx->counters.ptr + kSlotsKBase, scalars,
        (volatile unsigned long long*)ctx->pinned);
    DARBS_TRY(check_launch(ctx, "depth_histogram_kernel"));
    DARBS_CUDA_TRY(ctx, cudaEventRecord(ctx->k_ready, s));
    DARBS_CUDA_TRY(ctx, radix::launch_passes<unsigned>(dk0, or0, dk1, or1, (unsigned)n, depth_plan, ws.depth_tickets,
                                                       ws.depth_hist, ws.depth_status, s));
    ctx->launches += kDepthPasses;
    ctx->cur_order_buf = kDepthPasses & 1;
    const unsigned* order = ctx->cur_order_buf ? or1 : or0;

    unsigned long long k;
    const unsigned long long* k_dev = nullptr;
    if (ctx->entry_capacity > 0 && rects_done) {
        // the caller vouches for K <= capacity (darbs_cuda_set_entry_capacity): nothing of this view is
        // read back here, the kernels take K from the device and the host runs on; a view that breaks
        // the promise is truncated by expand_kernel and reported through the loss slot
        k = (unsigned long long)ctx->entry_capacity;
        k_dev = &scalars->total_entries;
    } else {
        // the host waits for K only (published before the depth sort): the GPU still has the sort
        // queued, so it does not idle while the rest of the iteration is being launched
        DARBS_CUDA_TRY(ctx, cudaEventSynchronize(ctx->k_ready));
        k = *(volatile unsigned long long*)ctx->pinned;
        if (k >= (1ull << 30)) return fail(ctx, DARBS_INVALID_PARAMETER, "more than 2^30 tile entries");
    }
    ctx->fwd_entries = (int64_t)k;
    if (k == 0) return DARBS_OK;

    // 2.-4. entries in depth order, stable sort on the tile, ranges
    if (ctx->tiles_x <= 256 && ctx->tiles_y <= 256)
        return tile_sort<unsigned short>(ctx, n, (int64_t)k, k_dev, order, rects, touched);
    return tile_sort<unsigned>(ctx, n, (int64_t)k, k_dev, order, rects, touched);
}

darbs_status export_bins(darbs_cuda_ctx* ctx, int64_t n, int32_t* tile_ranges, int32_t* point_list,
                         uint64_t* sort_keys, int32_t* depth_order) {
    cudaStream_t s = ctx->stream;
    const int tiles = ctx->tiles_x * ctx->tiles_y;
    const int64_t k = ctx->fwd_entries;
    if (tile_ranges && tiles)
        DARBS_CUDA_TRY(ctx, cudaMemcpyAsync(tile_ranges, ctx->ranges.ptr, sizeof(int2) * (size_t)tiles,
                                            cudaMemcpyDeviceToDevice, s));
    if (depth_order && n)
        DARBS_CUDA_TRY(ctx, cudaMemcpyAsync(depth_order, depth_order_ptr(ctx), sizeof(int32_t) * (size_t)n,
                                            cudaMemcpyDeviceToDevice, s));
    if (point_list && k)
        DARBS_CUDA_TRY(ctx, cudaMemcpyAsync(point_list, point_list_ptr(ctx), sizeof(int32_t) * (size_t)k,
                                            cudaMemcpyDeviceToDevice, s));
    if (sort_keys && k) {
        // rank_of[] reuses the inactive half of the order double buffer
        unsigned* or0 = (unsigned*)ctx->order.ptr;
        unsigned* rank_of = or0 + (size_t)(1 - ctx->cur_order_buf) * (ctx->order.bytes / 8);
        invert_order_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, depth_order_ptr(ctx), rank_of);
        DARBS_TRY(check_launch(ctx, "invert_order_kernel"));
        const unsigned* half = (const unsigned*)ctx->tile_keys.ptr + (size_t)ctx->cur_key_buf * (ctx->tile_keys.bytes / 8);
        if (ctx->tiles_x <= 256 && ctx->tiles_y <= 256)
            export_keys_kernel<unsigned short><<<grid_for(k, 256), 256, 0, s>>>(
                k, (const unsigned short*)half, ctx->tiles_x, (const unsigned*)point_list_ptr(ctx), rank_of,
                (unsigned long long*)sort_keys);
        else
            export_keys_kernel<unsigned><<<grid_for(k, 256), 256, 0, s>>>(
                k, half, ctx->tiles_x, (const unsigned*)point_list_ptr(ctx), rank_of, (unsigned long long*)sort_keys);
        DARBS_TRY(check_launch(ctx, "export_keys_kernel"));
    }
    return DARBS_OK;
}

}  // namespace darbs_b200
