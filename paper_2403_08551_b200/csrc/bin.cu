// a2. Tile binning with no depth key ("we can remove the sorting
// from rasterization"; north_star "duplicates (tile-id, gaussian-id) keys and
// radix-sorts them, with no depth key").
//
//   1. gauss_offset = exclusive scan of tiles_touched            (scan.cu)
//   2. duplicate: one (tile, gid) key per tile of each rectangle, row-major,
//      written warp-cooperatively (one warp walks 32 Gaussians; the lanes of
//      the warp write one Gaussian's keys in parallel -> coalesced, and one
//      huge Gaussian does not serialise a single thread)
//   3. stable LSD radix sort on the tile id only, ceil(log2(B*T)) bits in
//      passes of <= 8 bits; each pass = block digit histogram -> exclusive
//      scan of the digit-major [digit][chunk] table -> stable scatter, where
//      the in-chunk rank comes from __match_any_sync per 32-key stripe and
//      per-warp digit counters.  Hand-written, no CUB.
//   4. tile_range[t] = first index with key_tile >= t.
// Emission is in ascending gid, the sort is stable, so keys end in the unique
// lexicographic (tile, gid) order (reading R9) and match the oracle bit-exact.
#include "gi_internal.cuh"

namespace gi {
namespace {

constexpr int kRadixThreads = 256;
constexpr int kRadixWarps = kRadixThreads / 32;
constexpr int kRadixStripes = 16;                                // stripes of 32 per warp
constexpr int kChunk = kRadixThreads * kRadixStripes;            // 4096 keys per block
constexpr int kWarpSpan = kChunk / kRadixWarps;                  // 512 keys per warp

__device__ __forceinline__ int64_t eff_keys(const uint32_t* n_keys, int64_t cap) {
    int64_t k = (int64_t)*n_keys;
    return k < cap ? k : cap;
}

// ---------------------------------------------------------------- duplicate
__global__ void __launch_bounds__(256) duplicate_kernel(const Proj* __restrict__ proj,
                                                        const uint32_t* __restrict__ touched,
                                                        const uint32_t* __restrict__ offset,
                                                        int total, int n, int T, int TX,
                                                        int64_t cap, uint32_t* __restrict__ key_tile,
                                                        uint32_t* __restrict__ key_gid) {
    const int lane = threadIdx.x & 31;
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t cnt = 0, off = 0, tx0 = 0, tw = 1, ty0 = 0, tbase = 0;
    if (g < total) {
        cnt = touched[g];
        if (cnt) {
            off = offset[g];
            const float4 q1 = proj[g].q1;
            const float4 q2 = proj[g].q2;
            const uint32_t bx = __float_as_uint(q1.w), by = __float_as_uint(q2.w);
            tx0 = (bx & 0xffffu) / kTile;
            const uint32_t tx1 = (bx >> 16) / kTile;
            ty0 = (by & 0xffffu) / kTile;
            tw = tx1 - tx0 + 1;
            tbase = (uint32_t)(g / n) * (uint32_t)T;
        }
    }
    unsigned todo = __ballot_sync(kFull, cnt != 0);
    while (todo) {
        const int j = __ffs(todo) - 1;
        todo &= todo - 1;
        const uint32_t c = __shfl_sync(kFull, cnt, j);
        const uint32_t o = __shfl_sync(kFull, off, j);
        const uint32_t x0 = __shfl_sync(kFull, tx0, j);
        const uint32_t w = __shfl_sync(kFull, tw, j);
        const uint32_t y0 = __shfl_sync(kFull, ty0, j);
        const uint32_t tb = __shfl_sync(kFull, tbase, j);
        const uint32_t gid = (uint32_t)(g - lane + j);
        for (uint32_t i = lane; i < c; i += 32) {
            const int64_t pos = (int64_t)o + i;
            if (pos < cap) {
                const uint32_t ty = y0 + i / w, tx = x0 + i % w;
                key_tile[pos] = tb + ty * (uint32_t)TX + tx;
                key_gid[pos] = gid;
            }
        }
    }
}

// -------------------------------------------------------------- radix sort
__global__ void __launch_bounds__(kRadixThreads) radix_hist_kernel(const uint32_t* __restrict__ keys,
                                                                  const uint32_t* __restrict__ n_keys,
                                                                  int64_t cap, int shift, int bits,
                                                                  uint32_t* __restrict__ hist) {
    __shared__ uint32_t cnt[256];
    const int64_t K = eff_keys(n_keys, cap);
    const int64_t nc = (K + kChunk - 1) / kChunk;
    const int64_t b = blockIdx.x;
    if (b >= nc) return;
    const int R = 1 << bits;
    const uint32_t mask = (uint32_t)R - 1u;
    for (int i = threadIdx.x; i < R; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    const int64_t base = b * kChunk;
    for (int i = threadIdx.x; i < kChunk; i += blockDim.x) {
        const int64_t k = base + i;
        if (k < K) atomicAdd(&cnt[(keys[k] >> shift) & mask], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < R; d += blockDim.x) hist[(int64_t)d * nc + b] = cnt[d];
}

__global__ void __launch_bounds__(kRadixThreads) radix_scatter_kernel(
    const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
    uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
    const uint32_t* __restrict__ n_keys, int64_t cap, int shift, int bits,
    const uint32_t* __restrict__ hist_scanned) {
    __shared__ uint32_t whist[kRadixWarps][256];
    const int64_t K = eff_keys(n_keys, cap);
    const int64_t nc = (K + kChunk - 1) / kChunk;
    const int64_t b = blockIdx.x;
    if (b >= nc) return;
    const int R = 1 << bits;
    const uint32_t mask = (uint32_t)R - 1u;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kRadixWarps * 256; i += blockDim.x) (&whist[0][0])[i] = 0;
    __syncthreads();

    // Local stable ranks: warp w owns keys [base + w*512, +512) in 16 stripes.
    const int64_t wbase = b * kChunk + (int64_t)warp * kWarpSpan;
    uint32_t key[kRadixStripes], val[kRadixStripes], rank[kRadixStripes];
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int s = 0; s < kRadixStripes; ++s) {
        const int64_t k = wbase + s * 32 + lane;
        const bool valid = k < K;
        key[s] = valid ? keys_in[k] : 0u;
        val[s] = valid ? vals_in[k] : 0u;
        const unsigned act = __ballot_sync(kFull, valid);
        rank[s] = 0;
        if (valid) {
            const uint32_t d = (key[s] >> shift) & mask;
            const unsigned peers = __match_any_sync(act, d);
            const uint32_t before = whist[warp][d];
            rank[s] = before + __popc(peers & lt);
            __syncwarp(act);
            if ((peers & ~lt & ~(1u << lane)) == 0u)        // highest lane of the group
                whist[warp][d] = before + __popc(peers);
        }
        __syncwarp();
    }
    __syncthreads();
    // Cross-warp exclusive prefix per digit (warp order = key order).
    for (int d = threadIdx.x; d < R; d += blockDim.x) {
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < kRadixWarps; ++w) {
            const uint32_t c = whist[w][d];
            whist[w][d] = run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < kRadixStripes; ++s) {
        const int64_t k = wbase + s * 32 + lane;
        if (k < K) {
            const uint32_t d = (key[s] >> shift) & mask;
            const uint32_t dst = hist_scanned[(int64_t)d * nc + b] + whist[warp][d] + rank[s];
            keys_out[dst] = key[s];
            vals_out[dst] = val[s];
        }
    }
}

// ------------------------------------------------------------------ ranges
__global__ void __launch_bounds__(256) ranges_kernel(const uint32_t* __restrict__ key_tile,
                                                     const uint32_t* __restrict__ n_keys,
                                                     int64_t cap, uint32_t total_tiles,
                                                     uint32_t* __restrict__ range) {
    const int64_t K = eff_keys(n_keys, cap);
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > K) return;
    const int64_t prev = i > 0 ? (int64_t)key_tile[i - 1] : -1;
    const int64_t cur = i < K ? (int64_t)key_tile[i] : (int64_t)total_tiles;
    for (int64_t t = prev + 1; t <= cur; ++t) range[t] = (uint32_t)i;
}

struct BinWs {
    uint32_t* keys_a;
    uint32_t* vals_a;
    uint32_t* hist;
    uint32_t* scan_ws;
    size_t bytes;
};

int64_t max_chunks(int64_t cap) { return (cap + kChunk - 1) / kChunk; }

BinWs carve(void* base, int n, int64_t cap, const gi_frame& f) {
    const int64_t total = (int64_t)n * f.batch;
    const int64_t hist_words = max_chunks(cap) * 256;
    const int64_t scan_max = total + 1 > hist_words ? total + 1 : hist_words;
    char* p = static_cast<char*>(base);
    BinWs w;
    size_t off = 0;
    w.keys_a = reinterpret_cast<uint32_t*>(p + off); off += align_up(sizeof(uint32_t) * (size_t)cap);
    w.vals_a = reinterpret_cast<uint32_t*>(p + off); off += align_up(sizeof(uint32_t) * (size_t)cap);
    w.hist = reinterpret_cast<uint32_t*>(p + off); off += align_up(sizeof(uint32_t) * (size_t)hist_words);
    w.scan_ws = reinterpret_cast<uint32_t*>(p + off); off += align_up(sizeof(uint32_t) * scan_ws_words(scan_max));
    w.bytes = off;
    return w;
}

}  // namespace

size_t bin_ws_bytes(int n, int64_t cap, const gi_frame& f) { return carve(nullptr, n, cap, f).bytes; }

cudaError_t launch_bin(const Proj* proj, const uint32_t* tiles_touched, int n, const gi_frame& f,
                       int64_t cap, void* ws, uint32_t* gauss_offset, uint32_t* key_tile,
                       uint32_t* key_gid, uint32_t* tile_range, uint32_t* n_keys, cudaStream_t s) {
    BinWs w = carve(ws, n, cap, f);
    const int total = n * f.batch;
    const int T = tiles_x(f.width) * tiles_y(f.height);
    const uint32_t TT = (uint32_t)T * (uint32_t)f.batch;
    cudaError_t e;

    // 1. offsets (gauss_offset[total] = K, also copied to n_keys)
    e = scan_exclusive(tiles_touched, gauss_offset, total, nullptr, 1, w.scan_ws, n_keys, s);
    if (e != cudaSuccess) return e;
    // gauss_offset[total] = K: scan of a zero-extended input is not available,
    // so write it from n_keys
    e = cudaMemcpyAsync(gauss_offset + total, n_keys, sizeof(uint32_t), cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return e;

    // 2. radix plan: ceil(log2(TT)) key bits in passes of <= 8 bits
    int key_bits = 0;
    while ((1u << key_bits) < TT) ++key_bits;
    const int passes = (key_bits + 7) / 8;
    const int pass_bits = passes ? (key_bits + passes - 1) / passes : 0;
    // ping-pong so that the last pass lands in the caller's output
    uint32_t* bufk[2] = {w.keys_a, key_tile};
    uint32_t* bufv[2] = {w.vals_a, key_gid};
    int cur = (passes % 2 == 0) ? 1 : 0;       // emission buffer
    if (total > 0) {
        duplicate_kernel<<<(total + 255) / 256, 256, 0, s>>>(proj, tiles_touched, gauss_offset, total,
                                                             n, T, tiles_x(f.width), cap, bufk[cur],
                                                             bufv[cur]);
        note_launches(1);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    const int64_t nc_max = max_chunks(cap);
    for (int p = 0; p < passes; ++p) {
        const int shift = p * pass_bits;
        const int bits = (key_bits - shift) < pass_bits ? (key_bits - shift) : pass_bits;
        if (nc_max > 0) {
            radix_hist_kernel<<<(unsigned)nc_max, kRadixThreads, 0, s>>>(bufk[cur], n_keys, cap, shift,
                                                                         bits, w.hist);
            note_launches(1);
            if ((e = cudaGetLastError()) != cudaSuccess) return e;
        }
        e = scan_exclusive_spec(w.hist, w.hist, nc_max * (int64_t)(1 << bits), n_keys, kChunk,
                                1u << bits, cap, w.scan_ws, nullptr, s);
        if (e != cudaSuccess) return e;
        if (nc_max > 0) {
            radix_scatter_kernel<<<(unsigned)nc_max, kRadixThreads, 0, s>>>(
                bufk[cur], bufv[cur], bufk[cur ^ 1], bufv[cur ^ 1], n_keys, cap, shift, bits, w.hist);
            note_launches(1);
            if ((e = cudaGetLastError()) != cudaSuccess) return e;
        }
        cur ^= 1;
    }
    // 3. ranges over the sorted keys
    ranges_kernel<<<(unsigned)((cap + 1 + 255) / 256), 256, 0, s>>>(key_tile, n_keys, cap, TT,
                                                                   tile_range);
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace gi
