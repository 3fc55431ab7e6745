// Internal definitions shared by the libgi CUDA sources (sm_100a only).
// Nothing here is shared with the CPU oracle (oracle/).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <utility>

#include "../../include/gi.h"

// GI_ASSERT: device-side bounds checks compiled in only with -DGI_DEBUG (the
// pool's GPU boxes do not allow compute-sanitizer; the whole GPU test suite
// is run against a -DGI_DEBUG build instead: a violated check traps the
// kernel and fails the test).
#ifdef GI_DEBUG
#include <cassert>
#define GI_ASSERT(c) assert(c)
#else
#define GI_ASSERT(c) ((void)0)
#endif

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "libgi is written for sm_100a only"
#endif

namespace gi {

constexpr int kTile = 16;            // tile edge (R23)
constexpr int kTilePix = kTile * kTile;
constexpr int kWarps = 8;            // 256-thread CTA per tile, one pixel per thread
constexpr unsigned kFull = 0xffffffffu;

// sqrt(1/2 * log2(e)): sigma * log2(e) = (a dx)^2 + (b dx + c dy)^2 with
// (a, b, c) = kappa * (1/l1, -l2/(l1 l3), 1/l3)   [Sigma^-1 = L^-T L^-1]
constexpr double kKappa = 0.84932180028801907;   // sqrt(0.5 / ln 2)
constexpr double kLn2 = 0.69314718055994531;

// Projected Gaussian record, GI_PROJ_BYTES = 48, three float4.
//   q0 = {ix (int bits), iy (int bits), fx, fy}   centre = (ix + fx, iy + fy)
//   q1 = {a, b, c, bx}     factored conic; bx = x0 | x1 << 16 (u16 each)
//   q2 = {c'r, c'g, c'b, by}                    by = y0 | y1 << 16
// An empty box has x0 > x1 (0xffff0001 style: x0 = 1, x1 = 0).
struct __align__(16) Proj {
    float4 q0, q1, q2;
};
static_assert(sizeof(Proj) == GI_PROJ_BYTES, "record size");
// finalize / alloc read only the box words: q1.w (word 7) and q2.w (word 11)
static_assert(offsetof(Proj, q1) == 16 && offsetof(Proj, q2) == 32, "record layout");

constexpr uint32_t kEmptyBox = 1u;   // x0 = 1, x1 = 0

__host__ __device__ inline int tiles_x(int W) { return (W + kTile - 1) / kTile; }
__host__ __device__ inline int tiles_y(int H) { return (H + kTile - 1) / kTile; }

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Programmatic dependent launch (PDL): kernels of the fused chains are
// launched with programmatic stream serialization so that a kernel's launch
// and prologue overlap its predecessor's tail.  griddep_wait() must precede
// any access to memory the predecessor reads or writes; griddep_trigger()
// lets the successor be scheduled once every CTA of this grid has started.
// Both are no-ops for a normal launch.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }
// L2 prefetch: no data reaches the thread, so it is safe before
// griddep_wait() (L2 is the coherence point; a later load sees any write).
__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

bool use_pdl();   // default on; GI_NO_PDL=1 disables (A/B measurement)

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t s,
                       Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = use_pdl() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// launch_pdl with dynamic shared memory.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_smem(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = use_pdl() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// 64-bit integer add into a shared-memory (lo, hi) word pair by two native
// 32-bit atomics: exact mod 2^64 and order-independent like a 64-bit atomic
// add, without the compare-and-swap loop the compiler emits for 64-bit shared
// atomics (each wrap of the low word is seen as the carry of exactly one add).
__device__ __forceinline__ void shared_add_u64(uint32_t* pair, unsigned long long v) {
    const uint32_t lo = (uint32_t)v;
    uint32_t hi = (uint32_t)(v >> 32);
    if (lo != 0u) {
        const uint32_t old = atomicAdd(&pair[0], lo);
        hi += (uint32_t)(old + lo < old);
    }
    if (hi != 0u) atomicAdd(&pair[1], hi);
}

__device__ __forceinline__ unsigned long long shared_read_u64(const uint32_t* pair) {
    return (unsigned long long)pair[1] << 32 | pair[0];
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Contiguous partial slots per Gaussian: returns this lane's offset after a
// warp-aggregated atomic bump of *counter by cnt (all 32 lanes must call).
// The slot ORDER across Gaussians is arbitrary, but every value written to a
// slot and the order finalize sums a Gaussian's slots in are fixed, so the
// gradients are deterministic.
__device__ __forceinline__ uint32_t warp_alloc(uint32_t* counter, uint32_t cnt) {
    const int lane = threadIdx.x & 31;
    uint32_t x = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
    }
    uint32_t base = 0;
    if (lane == 31 && x > 0) base = atomicAdd(counter, x);
    base = __shfl_sync(kFull, base, 31);
    return base + x - cnt;
}

// Generic device scan (u32, exclusive) over `count` elements, count either a
// host constant or read from device memory.  Three launches, no inter-block
// waiting.  ws needs scan_ws_words(max_count) u32.
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTileElems = kScanThreads * kScanItems;   // 2048
size_t scan_ws_words(int64_t max_count);
// out may alias in.  count_dev: if non-null, count = *count_dev * count_mul
// (clamped to max_count).  total_out (device, may be null) receives the sum.
cudaError_t scan_exclusive(const uint32_t* in, uint32_t* out, int64_t max_count,
                           const uint32_t* count_dev, uint32_t count_mul, uint32_t* ws,
                           uint32_t* total_out, cudaStream_t s);
// count = ceil(min(*count_dev, cap) / div) * mul, clamped to max_count.
cudaError_t scan_exclusive_spec(const uint32_t* in, uint32_t* out, int64_t max_count,
                                const uint32_t* count_dev, uint32_t div, uint32_t mul, int64_t cap,
                                uint32_t* ws, uint32_t* total_out, cudaStream_t s);

// Per-thread count of kernels launched (or captured) through libgi; the
// bench reports it as gpu_launches.  Diagnostic only, never read by kernels.
void note_launches(int k);
int64_t g_launches_get();

// Internal launchers (api.cu validates arguments).
//
// Binning step 1 targets.  Every key (tile t, Gaussian g) is counted on
// tile_count[t] with an atomic that RETURNS the key's rank within the tile.
//  * direct binning (fused paths; slab != null): the key is written straight
//    to slab[t * slab_cap + rank] -- no scan, no scatter pass.  A tile whose
//    count exceeds slab_cap is served by its consumer from a stream of all
//    Gaussians instead (raster_common.cuh), so the result never depends on
//    the capacity.  Gaussians touching > 4 tiles are emitted warp-
//    cooperatively (post_project_warp) and get backward partial slots
//    allocated there.
//  * gi_bin contract (slab == null): ranks of <= 4-tile Gaussians are kept
//    in key_rank for the scatter; larger ones count on big_count.
// All counters must be zero on entry (bin_clear, or left zeroed by the
// consumer kernel of the previous fused call).
// tile_count words are kCountStride u32 apart: the count atomics (one per
// key, ~80 per tile, all issued within a few microseconds) then spread over
// L2 slices instead of queueing on the few slices that hold a packed table.
#ifndef GI_COUNT_STRIDE
#define GI_COUNT_STRIDE 8
#endif
constexpr int kCountStride = GI_COUNT_STRIDE;
// The frame paths (gi_render_frame, gi_decode_render_frame) on launches of
// fewer than kCountStrideWideTiles tiles (one C2-sized image) put the words
// 128 B apart instead: the few thousand counters then spread over more L2
// slices (C2 frame 56.2k -> 57.7k FPS, decode +2.7 %); the fit paths keep 32 B
// (-0.5 % at 128 B) and so do larger launches (C3 frame -4.7 % at 128 B).
// The workspace always has room for the wide layout, so both index the same
// allocation and the zero-fill rule is unchanged.
#ifndef GI_COUNT_STRIDE_WIDE
#define GI_COUNT_STRIDE_WIDE 32
#endif
constexpr int64_t kCountStrideWideTiles = 3072;
__host__ __device__ inline uint32_t count_alloc_stride(int64_t tiles) {
    return tiles < kCountStrideWideTiles ? (uint32_t)GI_COUNT_STRIDE_WIDE : (uint32_t)kCountStride;
}
__host__ __device__ inline uint32_t count_stride_for(int64_t tiles, bool frame = false) {
    return frame ? count_alloc_stride(tiles) : (uint32_t)kCountStride;
}

struct BinCounts {
    uint32_t* tile_count;   // [B*T * cstride] key counts (null: no counting)
    uint32_t* big_count;    // [B*T] gi_bin path: keys of Gaussians touching > 4 tiles
    uint4* key_rank;        // [B*N] gi_bin path: ranks of a small Gaussian's keys
    uint32_t* slab;         // direct binning: [B*T][slab_cap] key slots (null: gi_bin path)
    uint32_t slab_cap;
    uint32_t* n_keys_acc;   // direct binning: total keys accumulate here (may be null)
    uint32_t* gauss_off;    // direct binning + backward: partial slots of > 4-tile Gaussians
    uint32_t* alloc_counter;
    uint32_t part_cap;      // partial slots in all (4 total fixed + the allocatable rest)
    int row0, row1;         // NEXT-4 tile-row window [row0, row1); row1 = 0: whole image
    uint32_t cstride = kCountStride;   // u32 words between tile counts (count_stride_for)
};

// NEXT-4: a rank of a spatially sharded fit owns the tile rows [r0, r1).  A
// Gaussian's tile rectangle (x0, x1, y0, y1 in tiles) clipped to the window,
// rows made relative to r0; empty -> (0, -1, 0, -1).
__host__ __device__ inline int4 window_rect(int4 rect, int r0, int r1) {
    const int z = rect.z > r0 ? rect.z : r0, w = rect.w < r1 - 1 ? rect.w : r1 - 1;
    if (rect.x > rect.y || z > w) return make_int4(0, -1, 0, -1);
    return make_int4(rect.x, rect.y, z - r0, w - r0);
}
__host__ __device__ inline uint32_t rect_area(int4 r) {
    return (r.x > r.y || r.z > r.w) ? 0u : (uint32_t)((r.y - r.x + 1) * (r.w - r.z + 1));
}

// gauss_off value of a > 4-tile Gaussian whose slots did not fit: its tiles
// add their partial sums atomically into a per-Gaussian accumulator instead.
constexpr uint32_t kOffOverflow = 0xffffffffu;
// Backward partial slots: 4 per Gaussian + max(key capacity, 4 per Gaussian).
int64_t partial_cap(int n, int64_t cap, const gi_frame& f);

__device__ __forceinline__ uint32_t* count_word(const BinCounts& bc, int t) {
    return &bc.tile_count[(size_t)t * bc.cstride];
}

// Count the keys of Gaussian g (rect in tiles, `touched` tiles) into bc.
// Direct binning handles <= 4 tiles here, larger ones in post_project_warp.
__device__ __forceinline__ void count_keys(const BinCounts& bc, int g, int tx0, int tx1, int ty0,
                                           int ty1, uint32_t touched, int base, int TX) {
    if (touched <= 4u) {
        // key i -> tile (tx0 + i mod w, ty0 + i / w); the (up to) 4 atomics are
        // independent and issued back to back
        const int w = tx1 - tx0 + 1;
        uint32_t r[4] = {0u, 0u, 0u, 0u};
        int t[4] = {0, 0, 0, 0};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if ((uint32_t)i < touched) {
                const int dy = (i >= w) + (i >= 2 * w) + (i >= 3 * w);
                t[i] = base + (ty0 + dy) * TX + tx0 + (i - dy * w);
                GI_ASSERT(t[i] >= 0 && dy <= ty1 - ty0);
                r[i] = atomicAdd(count_word(bc, t[i]), 1u);
            }
        }
        if (bc.slab != nullptr) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if ((uint32_t)i < touched && r[i] < bc.slab_cap)
                    bc.slab[(size_t)t[i] * bc.slab_cap + r[i]] = (uint32_t)g;
        } else {
            bc.key_rank[g] = make_uint4(r[0], r[1], r[2], r[3]);
        }
    } else if (bc.slab == nullptr) {
        for (int ty = ty0; ty <= ty1; ++ty)
            for (int tx = tx0; tx <= tx1; ++tx) atomicAdd(&bc.big_count[base + ty * TX + tx], 1u);
    }
}

// Warp-uniform tail of a direct-binning producer (project_kernel, chained
// finalize): accumulate the key total, allocate backward partial slots for
// Gaussians touching > 4 tiles (4 total + offset; <= 4-tile Gaussians use
// the fixed slots 4 g ..) and emit their keys with the lanes of the warp
// striding over each one's tile rectangle.  touched = 0 for inactive lanes;
// rect = (tx0, tx1, ty0, ty1); base = image * T.
__device__ __forceinline__ void post_project_warp(const BinCounts& bc, uint32_t touched,
                                                  int4 rect, int g, int base, int TX, int total) {
    const int lane = threadIdx.x & 31;
    if (bc.n_keys_acc != nullptr) {
        const uint32_t sum = __reduce_add_sync(kFull, touched);
        if (lane == 0 && sum != 0u) atomicAdd(bc.n_keys_acc, sum);
    }
    if (bc.slab == nullptr) return;
    const bool big = touched > 4u;
    unsigned m = __ballot_sync(kFull, big);
    if (m == 0u) return;
    if (bc.gauss_off != nullptr) {
        const uint32_t off = warp_alloc(bc.alloc_counter, big ? touched : 0u);
        const uint64_t first = 4ull * (uint32_t)total + off;
        if (big) bc.gauss_off[g] = first + touched <= bc.part_cap ? (uint32_t)first : kOffOverflow;
    }
    // The warp's big Gaussians' keys as one flat list (exclusive scan of their
    // counts): lane l emits keys l, l + 32, ... of the list, so the rank
    // atomics of all of them are issued in ceil(total / 32) rounds instead of
    // one round trip per big Gaussian.  Owner of flat key f = the last lane
    // whose offset is <= f (binary search over the non-decreasing offsets;
    // lanes with no keys share the next owner's offset and come before it).
    const uint32_t c_l = big ? touched : 0u;
    uint32_t incl = c_l;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
    }
    const uint32_t off_l = incl - c_l;
    const uint32_t total_w = __shfl_sync(kFull, incl, 31);
    for (uint32_t f0 = 0; f0 < total_w; f0 += 32) {
        const uint32_t f = f0 + (uint32_t)lane;
        int j = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
            const uint32_t oj = __shfl_sync(kFull, off_l, j + step);
            if (oj <= f) j += step;
        }
        const int tx0 = __shfl_sync(kFull, rect.x, j), tx1 = __shfl_sync(kFull, rect.y, j);
        const int ty0 = __shfl_sync(kFull, rect.z, j);
        const int b = __shfl_sync(kFull, base, j);
        const uint32_t gid = (uint32_t)__shfl_sync(kFull, g, j);
        const uint32_t oj = __shfl_sync(kFull, off_l, j);
#ifdef GI_DEBUG
        const uint32_t cj = __shfl_sync(kFull, c_l, j);     // the owner's key count
#endif
        if (f < total_w) {
            const int i = (int)(f - oj), w = tx1 - tx0 + 1;
            GI_ASSERT(j >= 0 && j < 32 && i >= 0 && (uint32_t)i < cj);
            const int dy = i / w;
            const int t = b + (ty0 + dy) * TX + tx0 + (i - dy * w);
            const uint32_t r = atomicAdd(count_word(bc, t), 1u);
            if (r < bc.slab_cap) bc.slab[(size_t)t * bc.slab_cap + r] = gid;
        }
    }
}

// Optional fused outputs of the projection: step_counter is incremented once;
// counts: binning step 1 (see BinCounts).
struct ProjectFuse {
    uint32_t* step_counter;
    BinCounts counts;
};
// Direct-binning bookkeeping passed to the consumer tile kernels (all null on
// the gi_bin / tile_range paths): the consumer reads its count and slab,
// re-zeroes the count for the next call, and its CTA 0 resets the partial-
// slot allocator (close_segment).
struct ChainState {
    uint32_t* tile_count;
    uint32_t cstride = kCountStride;   // u32 words between tile counts (count_stride_for)
    uint32_t* alloc_counter;
    uint32_t* gauss_off;
    // direct binning (fused paths): the consumer reads its keys from the slab,
    // publishes *n_keys_acc to *n_keys and re-zeroes the accumulator
    uint32_t* slab;
    uint32_t slab_cap;
    uint32_t* n_keys;
    uint32_t* n_keys_acc;
    uint32_t* step_counter;   // chained fit: incremented once by the consumer
    // statistics (may be null): [0] tiles whose count exceeded the slab
    // (streamed from all Gaussians), [1] tiles whose segment exceeded the
    // kernel's sort buffer (rebuilt in order in global memory)
    uint32_t* seg_stats;
    int row0, row1;           // NEXT-4 tile-row window (row1 = 0: whole image)
    // fused Adam: the consumer's CTA 0 turns the step t (after the increment)
    // into {lr_t, 1 / (1 - b1^t), 1 / (1 - b2^t)} for the finalize kernel
    float* adam_consts;
    const uint32_t* step_read;
    float lr0;
    int half_every;
    float b1, b2;
    // fused Adan (NEXT-1): adan != 0 -> consts = {lr_t, 1/(1-b1^t), 1/(1-b2^t),
    // 1/sqrt(1-b3^t), 1 - lr_t wd, t == 1}
    int adan;
    float b3, wd;
};

// Optimiser arithmetic: the square root and the reciprocal of the update's
// denominator by MUFU (sqrt.approx, rcp.approx: within ~1 ulp each) instead
// of the IEEE sequences -- the update term then carries <= ~4e-7 relative
// error, inside c.4's 1e-6 bar on p (test_adam_step_nonzero_state_vs_oracle);
// m and v are exact fp32 FMAs as before.  One definition for every kernel
// (gi_adam_step, the fused finalize, the peer step, QAT; Adan likewise), so
// fused and standalone steps agree bit for bit.
__device__ __forceinline__ float sqrt_mufu(float x) {
    float r;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float rcp_mufu(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// One Adam update of a scalar (a5, reading R16): the arithmetic of
// gi_adam_step, shared with the fused finalize, the peer-exchange step
// (NEXT-4) and QAT so they all agree bit for bit.
__device__ __forceinline__ float adam_update(float& p, float g, float& m, float& v, float b1,
                                             float b2, float omb1, float omb2, float lr, float ibc1,
                                             float ibc2, float eps) {
    m = fmaf(b1, m, omb1 * g);
    v = fmaf(b2, v, omb2 * (g * g));
    const float mhat = m * ibc1;
    const float vhat = v * ibc2;
    p = p - (lr * mhat) * rcp_mufu(sqrt_mufu(vhat) + eps);
    return p;
}

// Adan step constants for step t (1-based), as the standalone adan_kernel and
// the fused finalize use them.
struct AdanConsts {
    float lr, ibc1, ibc2, isbc3, b1, b2, b3, eps, decay;
    int first;
};

// One Adan update of a scalar (NEXT-1, reading R28; see adan.cu):
//   d = g - g_prev (0 at t = 1); m = b1 m + (1-b1) g; v = b2 v + (1-b2) d;
//   n = b3 n + (1-b3) (g + b2 d)^2; g_prev = g;
//   p = p (1 - lr wd) - lr (m/(1-b1^t) + b2 v/(1-b2^t)) / (sqrt(n/(1-b3^t)) + eps)
__device__ __forceinline__ float adan1(float p, float g, float& m, float& v, float& n, float& gp,
                                       const AdanConsts& c) {
    const float d = c.first ? 0.0f : g - gp;
    m = fmaf(c.b1, m, (1.0f - c.b1) * g);
    v = fmaf(c.b2, v, (1.0f - c.b2) * d);
    const float u = fmaf(c.b2, d, g);
    n = fmaf(c.b3, n, (1.0f - c.b3) * (u * u));
    gp = g;
    const float upd = fmaf(c.b2 * c.ibc2, v, m * c.ibc1) * rcp_mufu(fmaf(sqrt_mufu(n), c.isbc3, c.eps));
    return fmaf(-c.lr, upd, p * c.decay);
}
cudaError_t launch_project(const float* params, int n, const gi_frame& f, uint32_t flags,
                           Proj* proj, uint32_t* tiles_touched, const ProjectFuse& fuse,
                           cudaStream_t s);
// gi_bin: count, scan, scatter and per-tile gid sort into contiguous arrays.
cudaError_t launch_bin(const Proj* proj, const uint32_t* tiles_touched, int n, const gi_frame& f,
                       int64_t cap, void* ws, uint32_t* key_tile, uint32_t* key_gid,
                       uint32_t* tile_range, uint32_t* n_keys, cudaStream_t s);
size_t bin_ws_bytes(int n, int64_t cap, const gi_frame& f);
BinCounts bin_counts(void* ws, int n, int64_t cap, const gi_frame& f);
// Direct binning (fused paths): keys go to slab = a key_gid array of cap
// entries, slab_cap = cap / (tiles x batch) per tile.
// Direct-binning slab per tile: cap / tiles, at least slab_min() keys (the
// slab array is slab_words() long, which may exceed cap: memory is plentiful,
// and a tile past its slab streams its keys from all N Gaussians).
// slab_min() = 1024, or GI_SLAB_MIN from the environment (tests force small
// slabs to exercise the streaming path; results never depend on it).
uint32_t slab_min();
// fused.cu: Gaussian-parallel tile kernels (default; GI_TILE3=0 -> round-1 kernels)
bool use_tile3();
bool use_render3(int tiles_per_launch, int n_per_image, int tiles_per_image);
cudaError_t launch_fused_backward(const Proj* proj, uint32_t* key_gid, const uint32_t* tile_range,
                                  const uint32_t* gauss_off, int n, const gi_frame& f,
                                  bool presorted, const float* dL_dimage, const float* target,
                                  float norm, int64_t pcap, float* partial, float* ovf,
                                  unsigned long long* sse_acc, float* image_out,
                                  const ChainState& cs, cudaStream_t s);
cudaError_t launch_fused_render(const Proj* proj, uint32_t* key_gid, const uint32_t* tile_range,
                                int n, const gi_frame& f, bool presorted, float* image,
                                const ChainState& cs, cudaStream_t s, bool decode = false);
uint32_t slab_capacity(int64_t cap, const gi_frame& f);
size_t slab_words(int64_t cap, const gi_frame& f);
uint32_t* bin_seg_stats(void* ws, int n, int64_t cap, const gi_frame& f);
// frame: the gi_render_frame / gi_decode_render_frame count layout (count_stride_for)
BinCounts bin_counts_direct(void* ws, int n, int64_t cap, const gi_frame& f, uint32_t* slab,
                            uint32_t* gauss_off, bool frame = false);
ChainState bin_chain_direct(void* ws, int n, int64_t cap, const gi_frame& f, uint32_t* slab,
                            uint32_t* gauss_off, uint32_t* n_keys, uint32_t* step_counter,
                            bool frame = false);
uint32_t* bin_alloc_counter(void* ws, int n, int64_t cap, const gi_frame& f);
cudaError_t bin_clear(void* ws, int n, int64_t cap, const gi_frame& f, cudaStream_t s);
cudaError_t launch_render(const Proj* proj, uint32_t* key_gid, const uint32_t* tile_range, int n,
                          const gi_frame& f, bool presorted, float* image, const ChainState& cs,
                          cudaStream_t s, bool decode = false);
size_t backward_ws_bytes(int n, int64_t cap, const gi_frame& f);
cudaError_t launch_backward(const float* params, const Proj* proj, const uint32_t* key_gid,
                            const uint32_t* tile_range, int n, const gi_frame& f, uint32_t flags,
                            const float* dL_dimage, const float* target, int64_t cap, void* ws,
                            float* grads, float* loss, float* image_out, cudaStream_t s);
cudaError_t launch_backward_alloc(const Proj* proj, int n, const gi_frame& f, int64_t cap, void* ws,
                                  cudaStream_t s);
float* backward_adam_consts(void* ws, int n, int64_t cap, const gi_frame& f);
uint32_t* backward_gauss_off(void* ws, int n, int64_t cap, const gi_frame& f);
cudaError_t launch_backward_tiles(const Proj* proj, uint32_t* key_gid, const uint32_t* tile_range,
                                  int n, const gi_frame& f, bool presorted,
                                  const float* dL_dimage, const float* target, int64_t cap,
                                  void* ws, float* image_out, const ChainState& cs,
                                  cudaStream_t s);
// Per-Gaussian reduction of the per-key partials + chain rule -> grads.  If
// adam_m is non-null the Adam update (device step counter) is fused in.
struct FusedAdam {
    float* params;
    float* m;
    float* v;
    const float* consts;      // {lr_t, 1 / (1 - b1^t), 1 / (1 - b2^t)} (ChainState.adam_consts)
    float b1, b2, eps;
    uint32_t* flag;
    // Adan instead of Adam (n != null): the third moment and the previous
    // gradient; consts as ChainState's Adan layout
    float* n;
    float* gprev;
    float b3;
    // chained fit step: project the updated Gaussian for the NEXT step (record,
    // tile count and binning step 1); null proj_out disables
    Proj* proj_out;
    uint32_t* touched_out;
    BinCounts counts;
    float k;
    uint32_t pos_flags;
};
// row0/row1: the NEXT-4 tile-row window the partials came from (row1 = 0:
// whole image).
cudaError_t launch_backward_finalize(const float* params, const Proj* proj, int n,
                                     const gi_frame& f, uint32_t flags, bool mse, int64_t cap,
                                     void* ws, float* grads, float* loss, const FusedAdam* adam,
                                     cudaStream_t s, int row0 = 0, int row1 = 0);
cudaError_t launch_adam(float* params, const float* grads, float* m, float* v, int64_t count,
                        int step, const uint32_t* step_dev, float lr, int half_every, float b1,
                        float b2, float eps, uint32_t* flag, cudaStream_t s);
cudaError_t launch_adan(float* params, const float* grads, float* m, float* v, float* n,
                        float* gprev, int64_t count, int step, const uint32_t* step_dev, float lr,
                        int half_every, float b1, float b2, float b3, float eps, float wd,
                        uint32_t* flag, cudaStream_t s);
struct QuantParams;
size_t qat_acc_words(int stages, int codebook);
cudaError_t launch_qat_quantize(const float* params, int n, const QuantParams& qp,
                                const float* qparams, const float* books, float* eff, void* acc,
                                uint32_t* step, float* consts, float lr, float b1, float b2,
                                cudaStream_t s);
cudaError_t launch_qat_update(float* params, float* m, float* v, float* grads, int n, int bits,
                              const float* qparams, const float* consts, float b1, float b2,
                              float eps, void* acc, int stages, int codebook, uint32_t* flag,
                              cudaStream_t s);
cudaError_t launch_qat_finish(float* qparams, float* qm, float* qv, float* books, float* ema_n,
                              float* ema_s, void* acc, int stages, int codebook, int n,
                              const float* consts, float b1, float b2, float eps, float decay,
                              float lambda, float* losses, cudaStream_t s);
cudaError_t launch_kmeans_step(const float* points, int n, int B, float* centroids,
                               uint32_t* assign, void* ws, cudaStream_t s);
cudaError_t launch_vq_encode(const float* params, bool logit, const gi_codec_meta& meta,
                             uint8_t* payload, float* eff, cudaStream_t s);
// NEXT-4 peer exchange: g = sum over r of grads[r] (rank order) then Adam;
// the n_loss floats after each rank's count gradients are summed into loss_out.
constexpr int kMaxPeers = 8;
cudaError_t launch_peer_adam(float* params, float* m, float* v, const float* const* grads, int G,
                             int64_t count, int step, float lr, float b1, float b2, float eps,
                             int n_loss, float* loss_out, uint32_t* flag, cudaStream_t s);
cudaError_t launch_vq_decode(const uint8_t* payload, const gi_codec_meta& meta, float* params,
                             cudaStream_t s);
// a6 + a1 fused (gi_decode_render_frame): decode record g and project it in
// one thread, direct binning as in launch_project; params_out may be null.
cudaError_t launch_decode_project(const uint8_t* payload, const gi_codec_meta& meta,
                                  float* params_out, const gi_frame& f, Proj* proj,
                                  uint32_t* tiles_touched, const ProjectFuse& fuse, cudaStream_t s);
cudaError_t launch_target_from_rgb8(const uint8_t* rgb, const gi_frame& f, float* target,
                                    cudaStream_t s);
cudaError_t launch_psnr(const float* image, const float* target, const gi_frame& f, float* psnr,
                        void* ws, cudaStream_t s);

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

__host__ __device__ inline bool pos_logit(uint32_t flags) { return (flags & GI_POS_NORMALIZED) == 0u; }
__host__ __device__ inline bool cov_rs(uint32_t flags) { return (flags & GI_COV_RS) != 0u; }
inline bool flags_valid(uint32_t flags) { return (flags & ~(GI_POS_NORMALIZED | GI_COV_RS)) == 0u; }

// Rotation-scaling covariance (Eq. 2-3) in fp64 with a fixed operation order
// (no contraction): Sigma = M M^T, M = R(theta) diag(s1e, s2e).
__device__ __forceinline__ void rs_sigma(double th, double s1e, double s2e, double S[3]) {
    const double c = cos(th), s = sin(th);
    const double m00 = __dmul_rn(c, s1e), m01 = __dmul_rn(-s, s2e);
    const double m10 = __dmul_rn(s, s1e), m11 = __dmul_rn(c, s2e);
    S[0] = __dadd_rn(__dmul_rn(m00, m00), __dmul_rn(m01, m01));
    S[1] = __dadd_rn(__dmul_rn(m00, m10), __dmul_rn(m01, m11));
    S[2] = __dadd_rn(__dmul_rn(m10, m10), __dmul_rn(m11, m11));
}

}  // namespace gi
