// Exclusive prefix sum over u32, used by binning when the tile count is too
// large for the one-CTA tile scan (batched launches).
// Reduce-then-scan: per-tile reduction, one-block scan of tile sums,
// per-tile downsweep.  No block ever waits on another (no look-back spin), so
// nothing can deadlock; the element count may live on the device (it is the
// data-dependent key count), grids are sized for the capacity and surplus
// blocks exit at once.
#include "gi_internal.cuh"

namespace gi {
namespace {

struct CountSpec {
    int64_t max_count;
    const uint32_t* count_dev;   // null -> max_count
    uint32_t div, mul;           // count = ceil(min(*count_dev, cap) / div) * mul
    int64_t cap;
};

__device__ __forceinline__ int64_t resolve_count(const CountSpec& c) {
    if (c.count_dev == nullptr) return c.max_count;
    int64_t k = (int64_t)*c.count_dev;
    if (k > c.cap) k = c.cap;
    int64_t v = (k + c.div - 1) / c.div * (int64_t)c.mul;
    return v < c.max_count ? v : c.max_count;
}

// Block-wide exclusive scan of one value per thread; returns the exclusive
// prefix and writes the block total to *total.
__device__ __forceinline__ uint32_t block_exclusive(uint32_t v, uint32_t* smem_warp, uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) smem_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < (int)(blockDim.x >> 5) ? smem_warp[lane] : 0u;
        uint32_t wx = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(kFull, wx, o);
            if (lane >= o) wx += y;
        }
        if (lane < (int)(blockDim.x >> 5)) smem_warp[lane] = wx - w;
        if (lane == 31) smem_warp[32] = wx;
    }
    __syncthreads();
    uint32_t r = smem_warp[warp] + x - v;
    *total = smem_warp[32];
    return r;
}

__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(const uint32_t* __restrict__ in,
                                                                  CountSpec cs,
                                                                  uint32_t* __restrict__ tile_sums) {
    __shared__ uint32_t sw[33];
    const int64_t count = resolve_count(cs);
    const int64_t base = (int64_t)blockIdx.x * kScanTileElems;
    if (base >= count) return;
    uint32_t s = 0;
    const int64_t i0 = base + (int64_t)threadIdx.x * kScanItems;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        int64_t i = i0 + j;
        if (i < count) s += in[i];
    }
    uint32_t tot;
    block_exclusive(s, sw, &tot);
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) scan_top_kernel(uint32_t* __restrict__ tile_sums, CountSpec cs,
                                                        uint32_t* __restrict__ total_out) {
    __shared__ uint32_t sw[33];
    const int64_t count = resolve_count(cs);
    const int64_t ntiles = (count + kScanTileElems - 1) / kScanTileElems;
    uint32_t carry = 0;
    for (int64_t base = 0; base < ntiles; base += blockDim.x) {
        int64_t i = base + threadIdx.x;
        uint32_t v = i < ntiles ? tile_sums[i] : 0u;
        uint32_t tot;
        uint32_t ex = block_exclusive(v, sw, &tot);
        if (i < ntiles) tile_sums[i] = carry + ex;
        carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0 && total_out != nullptr) *total_out = carry;
}

__global__ void __launch_bounds__(kScanThreads) scan_down_kernel(const uint32_t* __restrict__ in,
                                                                uint32_t* __restrict__ out,
                                                                CountSpec cs,
                                                                const uint32_t* __restrict__ tile_sums) {
    __shared__ uint32_t sw[33];
    const int64_t count = resolve_count(cs);
    const int64_t base = (int64_t)blockIdx.x * kScanTileElems;
    if (base >= count) return;
    const int64_t i0 = base + (int64_t)threadIdx.x * kScanItems;
    uint32_t v[kScanItems];
    uint32_t s = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        int64_t i = i0 + j;
        v[j] = i < count ? in[i] : 0u;
        s += v[j];
    }
    uint32_t tot;
    uint32_t run = block_exclusive(s, sw, &tot) + tile_sums[blockIdx.x];
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        int64_t i = i0 + j;
        if (i < count) out[i] = run;
        run += v[j];
    }
}

}  // namespace

size_t scan_ws_words(int64_t max_count) {
    return (size_t)((max_count + kScanTileElems - 1) / kScanTileElems) + 1;
}

cudaError_t scan_exclusive_spec(const uint32_t* in, uint32_t* out, int64_t max_count,
                                const uint32_t* count_dev, uint32_t div, uint32_t mul, int64_t cap,
                                uint32_t* ws, uint32_t* total_out, cudaStream_t s) {
    CountSpec cs{max_count, count_dev, div, mul, cap};
    const int64_t tiles = (max_count + kScanTileElems - 1) / kScanTileElems;
    if (tiles > 0) {
        scan_reduce_kernel<<<(unsigned)tiles, kScanThreads, 0, s>>>(in, cs, ws);
        note_launches(1);
    }
    scan_top_kernel<<<1, 1024, 0, s>>>(ws, cs, total_out);
    note_launches(1);
    if (tiles > 0) {
        scan_down_kernel<<<(unsigned)tiles, kScanThreads, 0, s>>>(in, out, cs, ws);
        note_launches(1);
    }
    return cudaGetLastError();
}

cudaError_t scan_exclusive(const uint32_t* in, uint32_t* out, int64_t max_count,
                           const uint32_t* count_dev, uint32_t count_mul, uint32_t* ws,
                           uint32_t* total_out, cudaStream_t s) {
    return scan_exclusive_spec(in, out, max_count, count_dev, 1, count_mul, max_count, ws,
                               total_out, s);
}

}  // namespace gi
