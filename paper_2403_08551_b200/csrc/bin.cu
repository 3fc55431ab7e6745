// a2. Tile binning with no depth key ("we can remove the sorting
// from rasterization"; north_star "duplicates (tile-id, gaussian-id) keys and
// radix-sorts them, with no depth key").
//
// The only order that matters is "grouped by tile" (R9); within a tile the
// keys are kept in ascending gid so the output is the unique lexicographic
// (tile, gid) order and the forward sum is deterministic.  On B200 the tile
// count of one image (1536 at 768x512) is tiny next to the key count, so the
// sort on the tile digit is done as ONE counting pass instead of LSD radix
// passes over 8-bit digits:
//
//   1. count    per-tile key counts (one RED per (Gaussian, tile)) -- fused
//               into the projection kernel on the fused paths
//   2. scan     tile_range = exclusive scan of the counts (one CTA when the
//               tile count is small; the 3-phase scan otherwise)
//   3. scatter  each (Gaussian, tile) key claims a slot in its tile's
//               segment with an atomic cursor: grouped by tile, gid order
//               inside a segment arbitrary
//   4. segsort  one CTA per tile restores ascending gid inside the segment:
//               rank sort (<= 256 keys), shared-memory bitonic sort
//               (<= 2048), or -- for a pathological segment -- a stable
//               in-order scan of all Gaussians of the image (no sort needed).
//               On the fused render / fit paths this step runs inside the
//               consumer tile kernel instead (same device function).
// Steps 1-3 are the counting (single-digit LSD radix) pass on the tile id;
// step 4 is the secondary key.  Hand-written, CUB-free, no data-dependent
// host sync: grids are sized by N, T or the key capacity.
#include "raster_common.cuh"

namespace gi {
namespace {

struct Rect {
    int tx0, tx1, ty0, ty1;
};

__device__ __forceinline__ Rect rect_of(const Proj& r) {
    const uint32_t bx = __float_as_uint(r.q1.w), by = __float_as_uint(r.q2.w);
    Rect q;
    q.tx0 = (int)(bx & 0xffffu) / kTile;
    q.tx1 = (int)(bx >> 16) / kTile;
    q.ty0 = (int)(by & 0xffffu) / kTile;
    q.ty1 = (int)(by >> 16) / kTile;
    return q;
}

// ------------------------------------------------------------------- count
__global__ void __launch_bounds__(256) count_kernel(const Proj* __restrict__ proj,
                                                    const uint32_t* __restrict__ touched, int total,
                                                    int n, int T, int TX, BinCounts bc) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    griddep_wait();
    griddep_trigger();
    if (g >= total) return;
    const uint32_t cnt = touched[g];
    if (cnt == 0) return;
    const Rect q = rect_of(proj[g]);
    count_keys(bc, g, q.tx0, q.tx1, q.ty0, q.ty1, cnt, (g / n) * T, TX);
}

// -------------------------------------------------------------------- scan
// One CTA: tile_range[0..TT] = exclusive scan of (tile_count + big_count),
// n_keys = total.  Range entries are clamped to the key capacity so that
// consumers never read past the key arrays when K > cap (n_keys still
// reports the true K).
__global__ void __launch_bounds__(1024) tile_scan_kernel(const uint32_t* __restrict__ tile_count,
                                                         const uint32_t* __restrict__ big_count,
                                                         int TT, int64_t cap,
                                                         uint32_t* __restrict__ tile_range,
                                                         uint32_t* __restrict__ n_keys) {
    __shared__ uint32_t warp_tot[32];
    __shared__ uint32_t carry_s;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    griddep_wait();
    griddep_trigger();
    const int per = (TT + blockDim.x - 1) / blockDim.x;       // consecutive items per thread
    const uint32_t cst = count_stride_for(TT);
    const int i0 = threadIdx.x * per;
    uint32_t s = 0;
    for (int k = 0; k < per; ++k) {
        const int i = i0 + k;
        if (i < TT) s += tile_count[(size_t)i * cst] + big_count[i];
    }
    uint32_t x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    if (warp == 0) {
        const uint32_t w = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0u;
        uint32_t wx = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, wx, o);
            if (lane >= o) wx += y;
        }
        warp_tot[lane] = wx - w;
        if (lane == 31) carry_s = wx;
    }
    __syncthreads();
    uint32_t run = warp_tot[warp] + x - s;
    for (int k = 0; k < per; ++k) {
        const int i = i0 + k;
        if (i < TT) {
            tile_range[i] = (int64_t)run < cap ? run : (uint32_t)cap;
            run += tile_count[(size_t)i * cst] + big_count[i];
        }
    }
    if (threadIdx.x == 0) {
        tile_range[TT] = (int64_t)carry_s < cap ? carry_s : (uint32_t)cap;
        *n_keys = carry_s;
    }
}

__global__ void combine_kernel(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                               uint32_t* __restrict__ out, int64_t count) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) out[i] = a[i * count_stride_for(count)] + b[i];
}

__global__ void clamp_kernel(uint32_t* __restrict__ v, int64_t count, int64_t cap) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count && (int64_t)v[i] > cap) v[i] = (uint32_t)cap;
}

// ----------------------------------------------------------------- scatter
// Slot of key (t, g): tile_start[t] + rank, where the rank of a small
// Gaussian's key was returned by its count atomic (key_rank), so the common
// case needs no atomic here; keys of Gaussians touching > 4 tiles follow the
// small ones (tile_start + tile_count) and claim a slot with an atomic on
// fill (handed to the whole warp when > 16 tiles).  With fuse_scan, every CTA
// first scans the (small) per-tile count tables itself into shared memory --
// a redundant 12 KB read per CTA instead of a separate launch -- and CTA 0
// publishes tile_range and n_keys.
constexpr int kFusedScanMax = 2048;

__global__ void __launch_bounds__(256) scatter_kernel(const Proj* __restrict__ proj,
                                                      const uint32_t* __restrict__ touched,
                                                      int total, int n, int T, int TX, int TT,
                                                      int64_t cap, bool fuse_scan, BinCounts bc,
                                                      uint32_t* __restrict__ tile_range,
                                                      uint32_t* __restrict__ n_keys,
                                                      uint32_t* __restrict__ fill,
                                                      uint32_t* __restrict__ key_tile,
                                                      uint32_t* __restrict__ key_gid) {
    __shared__ uint32_t start_s[kFusedScanMax];
    __shared__ uint32_t small_s[kFusedScanMax];
    __shared__ uint32_t wtot[kWarps];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    griddep_wait();
    griddep_trigger();
    // per-Gaussian inputs first: their latency overlaps the scan below
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t cnt = g < total ? touched[g] : 0u;
    Rect q{0, -1, 0, -1};
    uint4 rk = make_uint4(0u, 0u, 0u, 0u);
    if (cnt) {
        q = rect_of(proj[g]);
        if (cnt <= 4u) rk = bc.key_rank[g];
    }
    if (fuse_scan) {
        const int per = (TT + 255) / 256;                  // consecutive tiles per thread
        const int i0 = threadIdx.x * per;
        uint32_t sum = 0;
        for (int k = 0; k < per; ++k)
            if (i0 + k < TT) {
                const uint32_t sm = bc.tile_count[(size_t)(i0 + k) * bc.cstride];
                small_s[i0 + k] = sm;
                sum += sm + bc.big_count[i0 + k];
            }
        uint32_t x = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wtot[warp] = x;
        __syncthreads();
        uint32_t before = 0, all = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            before += w < warp ? wtot[w] : 0u;
            all += wtot[w];
        }
        uint32_t run = before + x - sum;
        for (int k = 0; k < per; ++k) {
            const int i = i0 + k;
            if (i < TT) {
                const uint32_t v = (int64_t)run < cap ? run : (uint32_t)cap;
                start_s[i] = v;
                if (blockIdx.x == 0) tile_range[i] = v;
                run += small_s[i] + bc.big_count[i];
            }
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            tile_range[TT] = (int64_t)all < cap ? all : (uint32_t)cap;
            *n_keys = all;
        }
        __syncthreads();
    }
    const int base = cnt ? (g / n) * T : 0;
    if (cnt > 0 && cnt <= 4) {
        const int w = q.tx1 - q.tx0 + 1;
        const uint32_t rks[4] = {rk.x, rk.y, rk.z, rk.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (i < (int)cnt) {
                const int t = base + (q.ty0 + i / w) * TX + q.tx0 + i % w;
                const uint32_t st = fuse_scan ? start_s[t] : tile_range[t];
                const int64_t slot = (int64_t)st + rks[i];
                if (slot < cap) {
                    key_tile[slot] = (uint32_t)t;
                    key_gid[slot] = (uint32_t)g;
                }
            }
        }
    } else if (cnt > 4 && cnt <= 16) {
        for (int ty = q.ty0; ty <= q.ty1; ++ty)
            for (int tx = q.tx0; tx <= q.tx1; ++tx) {
                const int t = base + ty * TX + tx;
                const uint32_t st = fuse_scan ? start_s[t] : tile_range[t];
                const uint32_t sm = fuse_scan ? small_s[t] : bc.tile_count[(size_t)t * bc.cstride];
                const int64_t slot = (int64_t)st + sm + atomicAdd(&fill[t], 1u);
                if (slot < cap) {
                    key_tile[slot] = (uint32_t)t;
                    key_gid[slot] = (uint32_t)g;
                }
            }
    }
    unsigned big = __ballot_sync(kFull, cnt > 16);
    while (big) {
        const int j = __ffs(big) - 1;
        big &= big - 1;
        const int tx0 = __shfl_sync(kFull, q.tx0, j), tx1 = __shfl_sync(kFull, q.tx1, j);
        const int ty0 = __shfl_sync(kFull, q.ty0, j);
        const uint32_t c = __shfl_sync(kFull, cnt, j);
        const int b = __shfl_sync(kFull, base, j);
        const int w = tx1 - tx0 + 1;
        const uint32_t gid = (uint32_t)(g - lane + j);
        for (uint32_t i = lane; i < c; i += 32) {
            const int t = b + (ty0 + (int)i / w) * TX + tx0 + (int)i % w;
            const uint32_t st = fuse_scan ? start_s[t] : tile_range[t];
            const uint32_t sm = fuse_scan ? small_s[t] : bc.tile_count[(size_t)t * bc.cstride];
            const int64_t slot = (int64_t)st + sm + atomicAdd(&fill[t], 1u);
            if (slot < cap) {
                key_tile[slot] = (uint32_t)t;
                key_gid[slot] = gid;
            }
        }
    }
}

// ----------------------------------------------------------------- segsort
// One CTA per tile: restore ascending gid inside the segment (see
// sorted_segment in raster_common.cuh) and write it back.
__global__ void __launch_bounds__(256) segsort_kernel(const Proj* __restrict__ proj, int n, int T,
                                                      int TX, const uint32_t* __restrict__ tile_range,
                                                      uint32_t* __restrict__ key_gid) {
    __shared__ alignas(16) uint32_t sl[kSortMax];
    __shared__ uint32_t scratch[kWarps];
    const int t = blockIdx.x;
    griddep_wait();
    griddep_trigger();
    const uint32_t s0 = tile_range[t], s1 = tile_range[t + 1];
    if (s1 - s0 <= 1) return;
    const int img = t / T, tl = t % T;
    const int cnt = sorted_segment(proj, key_gid, s0, s1, n, img, tl % TX, tl / TX, sl, scratch);
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) key_gid[s0 + i] = sl[i];
}

struct BinWs {
    uint32_t* tile_count;
    uint32_t* big_count;
    uint32_t* fill;
    uint32_t* alloc_counter;
    uint32_t* n_keys_acc;
    uint32_t* seg_stats;
    uint4* key_rank;
    uint32_t* scan_ws;
    size_t bytes;
};

BinWs carve(void* base, int n, int64_t cap, const gi_frame& f) {
    (void)cap;
    const int64_t TT = (int64_t)tiles_x(f.width) * tiles_y(f.height) * f.batch;
    const size_t total = (size_t)n * f.batch;
    char* p = static_cast<char*>(base);
    BinWs w;
    size_t off = 0;
    // tile_count (strided), big_count, fill and alloc_counter are adjacent: one memset
    w.tile_count = reinterpret_cast<uint32_t*>(p + off);
    off += sizeof(uint32_t) * (size_t)TT * count_alloc_stride(TT);
    w.big_count = reinterpret_cast<uint32_t*>(p + off); off += sizeof(uint32_t) * (size_t)TT;
    w.fill = reinterpret_cast<uint32_t*>(p + off); off += sizeof(uint32_t) * (size_t)TT;
    w.alloc_counter = reinterpret_cast<uint32_t*>(p + off); off += sizeof(uint32_t);
    w.n_keys_acc = reinterpret_cast<uint32_t*>(p + off); off += sizeof(uint32_t);
    w.seg_stats = reinterpret_cast<uint32_t*>(p + off); off += 2 * sizeof(uint32_t);
    off = align_up(off);                                   // 256-B (uint4 key_rank)
    w.key_rank = reinterpret_cast<uint4*>(p + off); off += align_up(sizeof(uint4) * (total + 1));
    w.scan_ws = reinterpret_cast<uint32_t*>(p + off); off += align_up(sizeof(uint32_t) * scan_ws_words(TT + 1));
    w.bytes = off;
    return w;
}

constexpr int64_t kOneCtaScanMax = 1 << 16;

}  // namespace

size_t bin_ws_bytes(int n, int64_t cap, const gi_frame& f) { return carve(nullptr, n, cap, f).bytes; }

BinCounts bin_counts(void* ws, int n, int64_t cap, const gi_frame& f) {
    BinWs w = carve(ws, n, cap, f);
    const int64_t TT = (int64_t)tiles_x(f.width) * tiles_y(f.height) * f.batch;
    BinCounts bc{w.tile_count, w.big_count, w.key_rank, nullptr, 0u, nullptr, nullptr, nullptr, 0u};
    bc.cstride = count_stride_for(TT);
    return bc;
}

uint32_t slab_min() {
    static const uint32_t v = [] {
        const char* e = std::getenv("GI_SLAB_MIN");
        return e == nullptr ? 1024u : (uint32_t)std::strtoul(e, nullptr, 10);
    }();
    return v;
}

uint32_t slab_capacity(int64_t cap, const gi_frame& f) {
    const int64_t TT = (int64_t)tiles_x(f.width) * tiles_y(f.height) * f.batch;
    if (TT <= 0) return 0u;
    const int64_t s = cap / TT, lo = (int64_t)slab_min();
    return (uint32_t)(s > lo ? s : lo);
}

size_t slab_words(int64_t cap, const gi_frame& f) {
    const size_t TT = (size_t)tiles_x(f.width) * tiles_y(f.height) * f.batch;
    return TT * slab_capacity(cap, f);
}

uint32_t* bin_seg_stats(void* ws, int n, int64_t cap, const gi_frame& f) {
    return carve(ws, n, cap, f).seg_stats;
}

BinCounts bin_counts_direct(void* ws, int n, int64_t cap, const gi_frame& f, uint32_t* slab,
                            uint32_t* gauss_off, bool frame) {
    BinWs w = carve(ws, n, cap, f);
    const int64_t pc = partial_cap(n, cap, f);
    BinCounts bc{w.tile_count, w.big_count, w.key_rank, slab, slab_capacity(cap, f),
                 w.n_keys_acc, gauss_off, gauss_off ? w.alloc_counter : nullptr,
                 (uint32_t)(pc < 0xffffffffll ? pc : 0xffffffffll)};
    bc.cstride = count_stride_for((int64_t)tiles_x(f.width) * tiles_y(f.height) * f.batch, frame);
    return bc;
}

ChainState bin_chain_direct(void* ws, int n, int64_t cap, const gi_frame& f, uint32_t* slab,
                            uint32_t* gauss_off, uint32_t* n_keys, uint32_t* step_counter,
                            bool frame) {
    BinWs w = carve(ws, n, cap, f);
    ChainState cs{};
    cs.tile_count = w.tile_count;
    cs.cstride = count_stride_for((int64_t)tiles_x(f.width) * tiles_y(f.height) * f.batch, frame);
    cs.alloc_counter = w.alloc_counter;
    cs.gauss_off = gauss_off;
    cs.slab = slab;
    cs.slab_cap = slab_capacity(cap, f);
    cs.n_keys = n_keys;
    cs.n_keys_acc = w.n_keys_acc;
    cs.seg_stats = w.seg_stats;
    cs.step_counter = step_counter;
    return cs;
}

uint32_t* bin_alloc_counter(void* ws, int n, int64_t cap, const gi_frame& f) {
    return carve(ws, n, cap, f).alloc_counter;
}

cudaError_t bin_clear(void* ws, int n, int64_t cap, const gi_frame& f, cudaStream_t s) {
    BinWs w = carve(ws, n, cap, f);
    const size_t TT = (size_t)tiles_x(f.width) * tiles_y(f.height) * f.batch;
    // tile_count .. n_keys_acc, seg_stats: adjacent
    return cudaMemsetAsync(w.tile_count, 0, sizeof(uint32_t) * ((count_alloc_stride(TT) + 2) * TT + 4), s);
}

cudaError_t launch_bin(const Proj* proj, const uint32_t* tiles_touched, int n, const gi_frame& f,
                       int64_t cap, void* ws, uint32_t* key_tile, uint32_t* key_gid,
                       uint32_t* tile_range, uint32_t* n_keys, cudaStream_t s) {
    BinWs w = carve(ws, n, cap, f);
    const int total = n * f.batch;
    const int TX = tiles_x(f.width);
    const int T = TX * tiles_y(f.height);
    const int TT = T * f.batch;
    cudaError_t e;
    if ((e = bin_clear(ws, n, cap, f, s)) != cudaSuccess) return e;
    if (total > 0) {
        e = launch_pdl(count_kernel, dim3((total + 255) / 256), dim3(256), s, proj, tiles_touched,
                       total, n, T, TX, BinCounts{w.tile_count, w.big_count, w.key_rank});
        if (e != cudaSuccess) return e;
        note_launches(1);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    const bool fuse = TT <= kFusedScanMax && total > 0;
    if (!fuse) {
        if (TT <= kOneCtaScanMax) {
            e = launch_pdl(tile_scan_kernel, dim3(1), dim3(1024), s, (const uint32_t*)w.tile_count,
                           (const uint32_t*)w.big_count, TT, cap, tile_range, n_keys);
            if (e != cudaSuccess) return e;
            note_launches(1);
        } else {
            combine_kernel<<<(TT + 255) / 256, 256, 0, s>>>(w.tile_count, w.big_count, tile_range, TT);
            note_launches(1);
            e = scan_exclusive(tile_range, tile_range, TT, nullptr, 1, w.scan_ws, n_keys, s);
            if (e != cudaSuccess) return e;
            e = cudaMemcpyAsync(tile_range + TT, n_keys, sizeof(uint32_t), cudaMemcpyDeviceToDevice, s);
            if (e != cudaSuccess) return e;
            clamp_kernel<<<(TT + 1 + 255) / 256, 256, 0, s>>>(tile_range, TT + 1, cap);
            note_launches(1);
        }
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    if (total > 0) {
        e = launch_pdl(scatter_kernel, dim3((total + 255) / 256), dim3(256), s, proj, tiles_touched,
                       total, n, T, TX, TT, cap, fuse, BinCounts{w.tile_count, w.big_count, w.key_rank},
                       tile_range, n_keys, w.fill, key_tile, key_gid);
        if (e != cudaSuccess) return e;
        note_launches(1);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    {   // per-tile gid order (the gi_bin contract)
        e = launch_pdl(segsort_kernel, dim3(TT), dim3(256), s, proj, n, T, TX,
                       (const uint32_t*)tile_range, key_gid);
        if (e != cudaSuccess) return e;
        note_launches(1);
    }
    return cudaGetLastError();
}

}  // namespace gi
