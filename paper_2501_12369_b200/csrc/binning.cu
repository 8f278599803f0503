// binning.cu — device restatement of darbs::bin_splats (reference
// src/rasterizer.cpp:25-53): global stable depth order, per-splat inclusive tile
// rectangle, per-tile depth-ordered index lists.
//
// Two-level sort instead of one wide (tile, depth) key:
//   1. stable LSD radix sort of the N (depth bits, index) pairs  -> depth order
//      (stability gives the reference's index tie-break, rasterizer.cpp:33);
//   2. tiles touched per splat, scanned IN DEPTH ORDER (read through the order by an input
//      iterator of the scan) -> write offsets;
//   3. every splat emits its (tile id, index) pairs at its offset, so the K
//      entries are already depth-ordered globally (a warp writes the entries of its 32
//      splats as one contiguous run);
//   4. stable radix sort of the K entries on the tile id bits only
//      (13 bits at 1080p: two 7-bit... passes) keeps depth order inside a tile;
//   5. tile ranges from the sorted tile ids.
// The tile rectangle is evaluated in FP64 on the float32 inputs so that
// floor((mu -+ R)/16) is decided on exactly the values the FP64 reference sees
// (rasterizer.cpp:40-45).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

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

// touched[] read through the depth order, so that the scan runs in depth order without a
// gathered copy of the counts (an input iterator of the scan).
struct TouchedInOrder {
    const unsigned* touched;
    const unsigned* order;
    __host__ __device__ unsigned operator()(unsigned r) const { return touched[order[r]]; }
};
using TouchedIter = thrust::transform_iterator<TouchedInOrder, thrust::counting_iterator<unsigned>>;

// K, the total of the per-splat tile counts (accumulated over kSlotsK addresses by the kernel
// that made the rectangles), goes to the device scalars and straight into pinned host memory
// (mapped under UVA): the host needs it to size the tile sort, and a write from the SM does not
// queue behind a bulk host <-> device copy that may be in flight on the copy engines.  It is
// known before the depth sort starts, so the host reads it while the GPU sorts.
__global__ void total_kernel(const unsigned long long* __restrict__ k_slots, Scalars* __restrict__ scalars,
                             volatile unsigned long long* host_total) {
    unsigned long long k = k_slots[threadIdx.x] + k_slots[threadIdx.x + 32];
    for (int o = 16; o > 0; o >>= 1) k += __shfl_xor_sync(0xffffffffu, k, o);
    if (threadIdx.x == 0) {
        scalars->total_entries = k;
        *host_total = k;
        __threadfence_system();
    }
}
static_assert(kSlotsK == 64, "total_kernel sums two slots per lane");

// TileKey: unsigned short while the tile ids fit 16 bits (every size of BASELINE.json does; 4K has
// 32 400 tiles), unsigned otherwise.  The tile sort then moves 6 bytes per entry and pass, not 8.
template <typename TileKey>
__global__ void __launch_bounds__(256)
duplicate_kernel(int64_t n, const unsigned* __restrict__ order, const unsigned* __restrict__ offsets,
                 const uint2* __restrict__ rects, const unsigned* __restrict__ touched, int tiles_x,
                 TileKey* __restrict__ tile_keys, unsigned* __restrict__ tile_vals) {
    // A warp takes 32 consecutive depth ranks and writes their entries TOGETHER: lane l owns the
    // splat of rank r0 + l, but entry e of the warp's run is written by lane e mod 32, which
    // finds the owning splat by a binary search over the lanes' offsets.  The writes of a warp
    // are then one contiguous run instead of 32 interleaved short ones (rasterizer.cpp:46-50).
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int64_t r0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) - lane;
    if (r0 >= n) return;
    const int64_t r = r0 + lane;
    unsigned idx = 0, cnt = 0, off = 0;
    uint2 rect = make_uint2(0, 0);
    if (r < n) {
        idx = order[r];
        rect = rects[idx];
        cnt = touched[idx];
        off = offsets[r];
    }
    const unsigned base = __shfl_sync(full, off, 0);
    // lanes past n inherit the end of the run, so that the search never lands on them
    const int last = (int)min((int64_t)31, n - 1 - r0);
    const unsigned end = __shfl_sync(full, off + cnt, last);
    const unsigned rel = (r < n ? off : end) - base;
    const unsigned total = end - base;
    for (unsigned e0 = 0; e0 < total; e0 += 32) {  // warp-uniform trip count: the shuffles need every lane
        const unsigned e = e0 + lane;
        int lo = 0;  // largest lane whose offset is <= e (zero-count lanes share the offset of the next)
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
            const unsigned probe = __shfl_sync(full, rel, min(lo + step, 31));
            if (lo + step <= 31 && probe <= e) lo += step;
        }
        const unsigned o_rel = __shfl_sync(full, rel, lo);
        const unsigned o_idx = __shfl_sync(full, idx, lo);
        const unsigned rx = __shfl_sync(full, rect.x, lo), ry = __shfl_sync(full, rect.y, lo);
        const unsigned x0 = rx & 0xffff, y0 = rx >> 16, w = (ry & 0xffff) - x0 + 1;
        if (e < total) {
            const unsigned q = e - o_rel;
            const unsigned qy = q / w, qx = q - qy * w;
            tile_keys[base + e] = (TileKey)((y0 + qy) * tiles_x + x0 + qx);
            tile_vals[base + e] = o_idx;
        }
    }
}

template <typename TileKey>
__global__ void ranges_kernel(int64_t k, const TileKey* __restrict__ sorted_tiles,
                              int2* __restrict__ ranges) {
    // eight consecutive entries per thread: one boundary test per entry against its predecessor
    constexpr int kPer = 8;
    const int64_t first = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * kPer;
    if (first >= k) return;
    unsigned prev = first > 0 ? (unsigned)sorted_tiles[first - 1] : 0xffffffffu;
    const int64_t stop = first + kPer < k ? first + kPer : k;
    for (int64_t i = first; i < stop; ++i) {
        const unsigned t = sorted_tiles[i];
        if (t != prev) {
            ranges[t].x = (int)i;
            if (prev != 0xffffffffu) ranges[prev].y = (int)i;
        }
        prev = t;
    }
    if (stop == k) ranges[prev].y = (int)k;
}

template <typename TileKey>
__global__ void export_keys_kernel(int64_t k, const TileKey* __restrict__ sorted_tiles,
                                   const unsigned* __restrict__ point_list,
                                   const unsigned* __restrict__ rank_of,
                                   unsigned long long* __restrict__ keys) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= k) return;
    keys[i] = ((unsigned long long)sorted_tiles[i] << 32) | rank_of[point_list[i]];
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

}  // namespace

const int32_t* point_list_ptr(const darbs_cuda_ctx* ctx) {
    return (const int32_t*)ctx->tile_vals.ptr + (size_t)ctx->cur_key_buf * (ctx->tile_vals.bytes / 8);
}
const uint32_t* depth_order_ptr(const darbs_cuda_ctx* ctx) {
    return (const uint32_t*)ctx->order.ptr + (size_t)ctx->cur_order_buf * (ctx->order.bytes / 8);
}

template <typename TileKey>
darbs_status tile_sort(darbs_cuda_ctx* ctx, int64_t n, int64_t k, int tiles, const unsigned* order,
                       const unsigned* offsets, const uint2* rects, const unsigned* touched) {
    cudaStream_t s = ctx->stream;
    // 3. duplicate in depth order
    DARBS_TRY(reserve(ctx, ctx->tile_keys, sizeof(unsigned) * 2 * (size_t)k));  // sized for 32-bit keys
    DARBS_TRY(reserve(ctx, ctx->tile_vals, sizeof(unsigned) * 2 * (size_t)k));
    TileKey* tk0 = (TileKey*)ctx->tile_keys.ptr;
    TileKey* tk1 = (TileKey*)((unsigned*)ctx->tile_keys.ptr + ctx->tile_keys.bytes / 8);
    unsigned* tv0 = (unsigned*)ctx->tile_vals.ptr;
    unsigned* tv1 = tv0 + ctx->tile_vals.bytes / 8;
    duplicate_kernel<TileKey><<<grid_for(n, 256), 256, 0, s>>>(n, order, offsets, rects, touched, ctx->tiles_x, tk0,
                                                      tv0);
    DARBS_TRY(check_launch(ctx, "duplicate_kernel"));

    // 4. stable sort on the tile bits
    cub::DoubleBuffer<TileKey> tkeys(tk0, tk1);
    cub::DoubleBuffer<unsigned> tvals(tv0, tv1);
    const int tbits = bits_for(tiles);
    size_t temp_bytes = 0;
    DARBS_CUDA_TRY(ctx, cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, tkeys, tvals, (int)k, 0,
                                                       tbits, s));
    DARBS_TRY(reserve(ctx, ctx->cub_temp, temp_bytes));
    temp_bytes = ctx->cub_temp.bytes;
    DARBS_CUDA_TRY(ctx, cub::DeviceRadixSort::SortPairs(ctx->cub_temp.ptr, temp_bytes, tkeys, tvals,
                                                       (int)k, 0, tbits, s));
    ctx->launches += 1 + (tbits + 7) / 8;
    ctx->cur_key_buf = tvals.Current() == tv0 ? 0 : 1;
    const TileKey* sorted_tiles = tkeys.Current();

    // 5. ranges
    ranges_kernel<TileKey><<<grid_for(((int64_t)k + 7) / 8, 256), 256, 0, s>>>((int64_t)k, sorted_tiles,
                                                            (int2*)ctx->ranges.ptr);
    return check_launch(ctx, "ranges_kernel");
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
    if (n >= (int64_t)1 << 31) return fail(ctx, DARBS_INVALID_PARAMETER, "too many splats");

    DARBS_TRY(reserve(ctx, ctx->ranges, sizeof(int2) * (size_t)(tiles > 0 ? tiles : 1)));
    DARBS_CUDA_TRY(ctx, cudaMemsetAsync(ctx->ranges.ptr, 0, sizeof(int2) * (size_t)tiles, s));
    Scalars* scalars = (Scalars*)((unsigned long long*)ctx->counters.ptr + 8);
    DARBS_CUDA_TRY(ctx, cudaMemsetAsync(ctx->counters.ptr, 0, sizeof(unsigned long long) * 10, s));
    unsigned long long* k_slots = (unsigned long long*)ctx->counters.ptr + kSlotsKBase;
    DARBS_CUDA_TRY(ctx, cudaMemsetAsync(k_slots, 0, sizeof(unsigned long long) * kSlotsK, s));
    ctx->fwd_entries = 0;
    ctx->cur_key_buf = 0;
    ctx->cur_order_buf = 0;
    if (sinks) *sinks = SplatSinks();
    if (n == 0 || tiles == 0) return DARBS_OK;

    const size_t nn = (size_t)n;
    DARBS_TRY(reserve(ctx, ctx->rects, sizeof(uint2) * nn + sizeof(unsigned) * nn));
    DARBS_TRY(reserve(ctx, ctx->depth_keys, sizeof(unsigned) * 2 * nn));
    DARBS_TRY(reserve(ctx, ctx->order, sizeof(unsigned) * 2 * nn));
    DARBS_TRY(reserve(ctx, ctx->offsets, sizeof(unsigned) * (nn + 1)));
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
    unsigned* offsets = (unsigned*)ctx->offsets.ptr;

    if (!rects_done) {
        rect_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, mu2, conic, radius, depth, valid, ctx->tiles_x,
                                                     ctx->tiles_y, rects, touched, dk0, or0, scalars,
                                                     (unsigned long long*)ctx->counters.ptr + kSlotsKBase);
        DARBS_TRY(check_launch(ctx, "rect_kernel"));
    }
    // K is complete: publish it now, and let the host pick it up while the depth sort runs
    DARBS_TRY(reserve_pinned(ctx, 64));
    total_kernel<<<1, 32, 0, s>>>((const unsigned long long*)ctx->counters.ptr + kSlotsKBase, scalars,
                                  (volatile unsigned long long*)ctx->pinned);
    DARBS_TRY(check_launch(ctx, "total_kernel"));
    DARBS_CUDA_TRY(ctx, cudaEventRecord(ctx->k_ready, s));

    // 1. stable depth sort
    cub::DoubleBuffer<unsigned> dkeys(dk0, dk1);
    cub::DoubleBuffer<unsigned> dvals(or0, or1);
    size_t temp_bytes = 0;
    DARBS_CUDA_TRY(ctx, cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, dkeys, dvals, (int)n, 0,
                                                       32, s));
    size_t scan_bytes = 0;
    DARBS_CUDA_TRY(ctx, cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, TouchedIter(thrust::counting_iterator<unsigned>(0u), TouchedInOrder{nullptr, nullptr}),
                                                     offsets, (int)n, s));
    DARBS_TRY(reserve(ctx, ctx->cub_temp, temp_bytes > scan_bytes ? temp_bytes : scan_bytes));
    temp_bytes = ctx->cub_temp.bytes;
    DARBS_CUDA_TRY(ctx, cub::DeviceRadixSort::SortPairs(ctx->cub_temp.ptr, temp_bytes, dkeys, dvals,
                                                       (int)n, 0, 32, s));
    ctx->launches += 5;  // onesweep: histogram + 4 digit passes
    const unsigned* order = dvals.Current();
    ctx->cur_order_buf = order == or0 ? 0 : 1;

    // 2. offsets in depth order, total K
    TouchedIter in_order(thrust::counting_iterator<unsigned>(0u), TouchedInOrder{touched, order});
    scan_bytes = ctx->cub_temp.bytes;
    DARBS_CUDA_TRY(ctx, cub::DeviceScan::ExclusiveSum(ctx->cub_temp.ptr, scan_bytes, in_order, offsets, (int)n, s));
    ctx->launches += 2;
    // the host waits for K only (published before the depth sort): the GPU still has the sort and
    // the scan queued, so it does not idle while the rest of the iteration is being launched
    DARBS_CUDA_TRY(ctx, cudaEventSynchronize(ctx->k_ready));
    const unsigned long long k = *(volatile unsigned long long*)ctx->pinned;
    if (k >= (1ull << 31)) return fail(ctx, DARBS_INVALID_PARAMETER, "more than 2^31 tile entries");
    ctx->fwd_entries = (int64_t)k;
    if (k == 0) return DARBS_OK;

    // 3.-5. duplicate in depth order, stable sort on the tile bits, ranges
    if (tiles <= 65536)
        return tile_sort<unsigned short>(ctx, n, (int64_t)k, tiles, order, offsets, rects, touched);
    return tile_sort<unsigned>(ctx, n, (int64_t)k, tiles, order, offsets, rects, touched);
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
        if (tiles <= 65536)
            export_keys_kernel<unsigned short><<<grid_for(k, 256), 256, 0, s>>>(
                k, (const unsigned short*)half, (const unsigned*)point_list_ptr(ctx), rank_of,
                (unsigned long long*)sort_keys);
        else
            export_keys_kernel<unsigned><<<grid_for(k, 256), 256, 0, s>>>(
                k, half, (const unsigned*)point_list_ptr(ctx), rank_of, (unsigned long long*)sort_keys);
        DARBS_TRY(check_launch(ctx, "export_keys_kernel"));
    }
    return DARBS_OK;
}

}  // namespace darbs_b200
