// Tile rasteriser building blocks shared by the forward (render.cu), the
// fused forward + L2 + backward (backward.cu) and the binning (bin.cu)
// kernels.
//
// CTA = one 16x16 tile of one image, 256 threads, one pixel per thread.
// Warp w covers an 8x4 pixel block (w & 1 -> x half, w >> 1 -> y quarter), so
// a warp skips a Gaussian whose box misses its block (warp culling): at the
// paper's init scale this evaluates ~3x fewer pairs than whole-tile
// evaluation.  The two-pixel kernels (render2_kernel,
// backward_tile2_kernel) use 128 threads and 8x8 warp blocks instead; the
// segment helpers below take the CTA size (NT) and sort-buffer size (SMAX)
// as template parameters.
//
// The tile's key segment is first brought into ascending-gid order in shared
// memory (direct binning leaves it in atomic order), then, per batch of up to
// kBatch keys, each thread stages one record converted to TILE-LOCAL
// coordinates (StagedRecords below: conic + colour, centre minus the tile
// origin -- ix - tx0 is an exact small integer, + fx rounds once -- and the
// box clipped to the tile).  Each warp then compacts the batch into its own
// candidate list: the record index + the 32-bit mask of its lanes whose pixel
// lies in the box, so the inner loop needs no bit scanning and a
// one-instruction box test.  The box is staged as 16-bit column / row masks of
// the tile, so a warp's 32-lane mask is two bit-field extracts and two
// multiplies.
#pragma once
#include "gi_internal.cuh"

namespace gi {

constexpr int kSortMax = 2048;      // segments sorted in shared memory (8 KB)
constexpr int kRankMax = 256;       // rank sort up to this size, bitonic above
#ifndef GI_BATCH
#define GI_BATCH 128
#endif
constexpr int kBatch = GI_BATCH;    // records staged per batch (<= 256)

struct TileCtx {
    int img, tile, tx, ty;        // tile coordinates
    int lane, warp;
    int x, y;                     // global pixel of this thread
    float cx, cy;                 // tile-local pixel centre (x + 1/2 - 16 tx)
    int wx0, wy0;                 // warp block origin (global pixels)
    int csh, rsh;                 // warp block: column / row shift in the tile masks
    int row0, row1;               // tile-row window of the launch (NEXT-4); tile = relative index
    bool in_image;
};

// Grid: (tiles_x, window rows, images) -- no integer division per CTA.  The
// CTA's tile row is row0 + blockIdx.y; `tile` indexes the window.
__device__ __forceinline__ TileCtx make_tile_ctx(int W, int H, int TX, int row0) {
    TileCtx c;
    c.tx = blockIdx.x;
    c.ty = row0 + blockIdx.y;
    c.img = blockIdx.z;
    c.tile = blockIdx.y * TX + c.tx;
    c.row0 = row0;
    c.row1 = row0 + gridDim.y;
    c.lane = threadIdx.x & 31;
    c.warp = threadIdx.x >> 5;
    // thread bits: [0,3) column in the block, [3,5) row, [5] x half, [6,8) y quarter
    const int lx = (int)((threadIdx.x & 7u) | ((threadIdx.x >> 2) & 8u));
    const int ly = (int)(((threadIdx.x >> 3) & 3u) | ((threadIdx.x >> 4) & 12u));
    c.x = c.tx * kTile + lx;
    c.y = c.ty * kTile + ly;
    c.cx = (float)lx + 0.5f;
    c.cy = (float)ly + 0.5f;
    c.wx0 = c.tx * kTile + (c.warp & 1) * 8;
    c.wy0 = c.ty * kTile + (c.warp >> 1) * 4;
    c.csh = (c.warp & 1) * 8;
    c.rsh = (c.warp >> 1) * 4;
    c.in_image = c.x < W && c.y < H;
    return c;
}

// Staged record j (tile-local):
//   a = {a, b, c, c'r}          factored conic (sigma log2 e = (a dx)^2 + (b dx + c dy)^2)
//   b = {c'g, c'b, mx, my}      centre minus the tile origin, rounded to fp32
//   o = {u0, v0}                the rounding of (mx, my) carried into (u, v):
//                               u = a dx + u0, v = b dx + c dy + v0 with
//                               dx = cx - mx, u0 = -a mx_lo, v0 = -(b mx_lo + c my_lo)
//   c = {lx0 | lx1 << 8 | ly0 << 16 | ly1 << 24   box clipped to the tile,
//        column mask | row mask << 16,            the same as 16-bit masks,
//        partial slot (backward only), gid}
// Why o: a tile-local centre rounds to ulp(|mx|) (~5e-7 px at |mx| ~ 10),
// and the conic multiplies that by a (or b) -- ~70 px^-1 for a Gaussian
// 0.012 px wide, enough to move sigma by 1e-4 and its gradient past the 1e-4
// bar.  With the exact remainder mx_lo folded into (u0, v0), (u, v) carry an
// error of ulp(dx) instead, at no extra instruction per pair (u, v become
// FMAs with the correction as addend).
template <int NB>
struct StagedRecordsN {
    static constexpr int kN = NB;
    float4 a[NB];
    float4 b[NB];
    float2 o[NB];
    uint4 c[NB];
};
using StagedRecords = StagedRecordsN<kBatch>;

// Per-warp compacted candidate list for one batch: (record index, lane mask).
struct WarpLists {
    uint2 ent[kWarps][kBatch];
    int cnt[kWarps];
};

__device__ __forceinline__ uint32_t span_mask16(int lo, int hi) {
    return ((2u << hi) - 1u) & ~((1u << lo) - 1u);
}

// Stage record j = threadIdx.x (j < cnt) for gid into shared memory.  With
// gauss_off (backward), also the Gaussian's partial slot for this tile: its
// contiguous range (4 gid, or gauss_off[gid] above 4 tiles) + the rank of this tile in its tile
// rectangle (row-major), the order finalize sums in.
template <class SR>
__device__ __forceinline__ void stage_gid(SR& sr, const Proj* __restrict__ proj,
                                          uint32_t gid, int j, const TileCtx& t,
                                          const uint32_t* __restrict__ gauss_off = nullptr) {
    const Proj r = proj[gid];
    const int tx0 = t.tx * kTile, ty0 = t.ty * kTile;
    const int ix = __float_as_int(r.q0.x), iy = __float_as_int(r.q0.y);
    // (ix - tx0) + fx as mx + mx_lo exactly (TwoSum; the integer is exact in fp32)
    const float ixf = (float)(ix - tx0), iyf = (float)(iy - ty0);
    const float mx = __fadd_rn(ixf, r.q0.z), my = __fadd_rn(iyf, r.q0.w);
    const float bx_ = __fsub_rn(mx, ixf), by_ = __fsub_rn(my, iyf);
    const float mx_lo = __fadd_rn(__fsub_rn(ixf, __fsub_rn(mx, bx_)), __fsub_rn(r.q0.z, bx_));
    const float my_lo = __fadd_rn(__fsub_rn(iyf, __fsub_rn(my, by_)), __fsub_rn(r.q0.w, by_));
    const uint32_t bx = __float_as_uint(r.q1.w), by = __float_as_uint(r.q2.w);
    const int x0 = (int)(bx & 0xffffu), x1 = (int)(bx >> 16);
    const int y0 = (int)(by & 0xffffu), y1 = (int)(by >> 16);
    const int lx0 = max(x0 - tx0, 0), lx1 = min(x1 - tx0, kTile - 1);
    const int ly0 = max(y0 - ty0, 0), ly1 = min(y1 - ty0, kTile - 1);
    uint32_t slot = 0;
    if (gauss_off != nullptr) {
        // slots 4 gid.. for Gaussians touching <= 4 tiles of the window, the
        // rank of this tile in the (window-clipped) rectangle, row-major
        const int4 rw = window_rect(make_int4(x0 / kTile, x1 / kTile, y0 / kTile, y1 / kTile),
                                    t.row0, t.row1);
        const uint32_t off = rect_area(rw) <= 4u ? 4u * gid : gauss_off[gid];
        slot = off == kOffOverflow
                   ? kOffOverflow
                   : off + (uint32_t)((t.ty - t.row0 - rw.z) * (rw.y - rw.x + 1) + (t.tx - rw.x));
    }
    // a staged record overlaps the tile (its key is in the tile's list)
    GI_ASSERT(j >= 0 && j < SR::kN && lx0 <= lx1 && ly0 <= ly1);
    sr.a[j] = make_float4(r.q1.x, r.q1.y, r.q1.z, r.q2.x);
    sr.b[j] = make_float4(r.q2.y, r.q2.z, mx, my);
    sr.o[j] = make_float2(-(r.q1.x * mx_lo), -fmaf(r.q1.y, mx_lo, r.q1.z * my_lo));
    sr.c[j] = make_uint4((uint32_t)(lx0 | lx1 << 8 | ly0 << 16 | ly1 << 24),
                         span_mask16(lx0, lx1) | span_mask16(ly0, ly1) << 16, slot, gid);
}

// Lanes of the 8x4 warp block (lane = ly * 8 + lx) inside the box given by
// its 16-bit tile column / row masks: the block's 8 columns replicated into
// the bytes of its 4 set rows (bit i of the row nibble -> bit 8 i).
__device__ __forceinline__ uint32_t warp_box_mask(uint32_t masks, const TileCtx& t) {
    const uint32_t cols = (masks >> t.csh) & 0xffu;
    const uint32_t rows = (masks >> (16 + t.rsh)) & 0xfu;
    return ((rows * 0x00204081u) & 0x01010101u) * cols;
}

// Build this warp's candidate list for a staged batch of cnt records.
__device__ __forceinline__ int build_warp_list(const StagedRecords& sr, WarpLists& wl, int cnt,
                                               const TileCtx& t) {
    int n = 0;
    for (int q = 0; q < cnt; q += 32) {
        const int j = q + t.lane;
        const uint32_t m = j < cnt ? warp_box_mask(sr.c[j].y, t) : 0u;
        const unsigned hit = __ballot_sync(kFull, m != 0u);
        if (m != 0u) wl.ent[t.warp][n + __popc(hit & lanemask_lt())] = make_uint2((uint32_t)j, m);
        n += __popc(hit);
    }
    __syncwarp();
    return n;
}

// exp(-sigma) for the staged record (factored conic, MUFU.EX2), and the
// scaled offsets u = a dx, v = b dx + c dy (sigma log2 e = u^2 + v^2).
struct PairEval {
    float w, u, v;
};

__device__ __forceinline__ PairEval eval_pair(const float4 A, const float4 B, const float2 O,
                                              const TileCtx& t) {
    PairEval e;
    const float dx = t.cx - B.z;
    const float dy = t.cy - B.w;
    e.u = fmaf(A.x, dx, O.x);
    e.v = fmaf(A.y, dx, fmaf(A.z, dy, O.y));
    e.w = ex2_approx(fmaf(-e.u, e.u, -(e.v * e.v)));
    return e;
}

// Accumulate Eq. 7 for this thread's pixel over the warp's candidate list
// (ascending record index = ascending gid).
__device__ __forceinline__ void forward_batch(const StagedRecords& sr, const WarpLists& wl, int n,
                                              const TileCtx& t, float& acc0, float& acc1,
                                              float& acc2) {
    const uint2* ent = wl.ent[t.warp];
    const uint32_t bit = 1u << t.lane;
#pragma unroll 2
    for (int k = 0; k < n; ++k) {
        const uint2 en = ent[k];
        const float4 A = sr.a[en.x];
        const float4 B = sr.b[en.x];
        const PairEval pe = eval_pair(A, B, sr.o[en.x], t);
        const float w = (en.y & bit) ? pe.w : 0.f;
        acc0 = fmaf(A.w, w, acc0);
        acc1 = fmaf(B.x, w, acc1);
        acc2 = fmaf(B.y, w, acc2);
    }
}

// ----------------------------------------------------- segment ordering
// Bring the tile's key segment [s, e) into ascending gid order.  Returns the
// segment length if it now sits sorted in `sl` (shared, kSortMax entries), or
// -1 if it was longer than kSortMax and was rebuilt IN ORDER directly in the
// global key_gid segment (stable scan of all Gaussians of the image).
// Gids within a segment are distinct.  All threads of the CTA must call.
__device__ __forceinline__ bool covers_tile(const Proj* __restrict__ proj, uint32_t g, int tx,
                                            int ty) {
    const uint32_t bx = __float_as_uint(proj[g].q1.w), by = __float_as_uint(proj[g].q2.w);
    const int x0 = (int)(bx & 0xffffu), x1 = (int)(bx >> 16);
    const int y0 = (int)(by & 0xffffu), y1 = (int)(by >> 16);
    return x0 <= x1 && y0 <= y1 && x0 / kTile <= tx && x1 / kTile >= tx && y0 / kTile <= ty &&
           y1 / kTile >= ty;
}

// r - #{v.x, v.y, v.z, v.w < mine}: the borrow of v - mine is the compare,
// subtracted straight from r (2 instructions per compare instead of 3).
__device__ __forceinline__ uint32_t count_below4(const uint4 v, uint32_t mine, uint32_t r) {
    asm("{\n\t.reg .u32 t;\n\t"
        "sub.cc.u32 t, %1, %5;\n\tsubc.u32 %0, %0, 0;\n\t"
        "sub.cc.u32 t, %2, %5;\n\tsubc.u32 %0, %0, 0;\n\t"
        "sub.cc.u32 t, %3, %5;\n\tsubc.u32 %0, %0, 0;\n\t"
        "sub.cc.u32 t, %4, %5;\n\tsubc.u32 %0, %0, 0;\n\t}"
        : "+r"(r)
        : "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(mine));
    return r;
}

// NT = threads per CTA (256, or 128 for the two-pixel render kernel): each
// thread ranks kRankMax / NT of the keys.
template <int NT = 256, int SMAX = kSortMax>
__device__ __forceinline__ int sorted_segment(const Proj* __restrict__ proj,
                                              uint32_t* __restrict__ key_gid, uint32_t s,
                                              uint32_t e, int n, int img, int tx, int ty,
                                              uint32_t* sl, uint32_t* scratch8) {
    constexpr int E = kRankMax / NT;
    const int cnt = (int)(e - s);
    if (cnt <= kRankMax) {
        uint32_t mine[E];
#pragma unroll
        for (int q = 0; q < E; ++q) {
            const int i = (int)threadIdx.x + q * NT;
            mine[q] = i < cnt ? key_gid[s + i] : 0xffffffffu;
            sl[i] = mine[q];
        }
        __syncthreads();
        uint32_t r[E];   // entries >= cnt hold 0xffffffff and never count
#pragma unroll
        for (int q = 0; q < E; ++q) {
            r[q] = 0u;
            if ((int)threadIdx.x + q * NT < cnt) {
                const uint4* s4 = reinterpret_cast<const uint4*>(sl);
                for (int k = 0; k < (cnt + 3) >> 2; ++k) r[q] = count_below4(s4[k], mine[q], r[q]);
            }
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < E; ++q)
            if ((int)threadIdx.x + q * NT < cnt) {
                GI_ASSERT((0u - r[q]) < (uint32_t)cnt);
                sl[0u - r[q]] = mine[q];
            }
        __syncthreads();
        return cnt;
    }
    if (cnt <= SMAX) {
        int P = 512;
        while (P < cnt) P <<= 1;
        for (int i = threadIdx.x; i < P; i += blockDim.x) sl[i] = i < cnt ? key_gid[s + i] : 0xffffffffu;
        __syncthreads();
        for (int k = 2; k <= P; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = threadIdx.x; i < P; i += blockDim.x) {
                    const int l = i ^ j;
                    if (l > i) {
                        const uint32_t a = sl[i], b = sl[l];
                        if ((a > b) == ((i & k) == 0)) {
                            sl[i] = b;
                            sl[l] = a;
                        }
                    }
                }
                __syncthreads();
            }
        }
        return cnt;
    }
    // pathological segment: stable in-order rebuild in global memory
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t out = 0;
    for (int base = 0; base < n; base += blockDim.x) {
        const int g = base + threadIdx.x;
        const bool hit = g < n && covers_tile(proj, (uint32_t)(img * n + g), tx, ty);
        const unsigned m = __ballot_sync(kFull, hit);
        if (lane == 0) scratch8[warp] = __popc(m);
        __syncthreads();
        uint32_t before = 0, tot = 0;
        for (int w = 0; w < NT / 32; ++w) {
            before += w < warp ? scratch8[w] : 0u;
            tot += scratch8[w];
        }
        if (hit) {
            const uint32_t slot = s + out + before + __popc(m & lanemask_lt());
            if (slot < e) key_gid[slot] = (uint32_t)(img * n + g);
        }
        out += tot;
        __syncthreads();
    }
    __threadfence_block();
    __syncthreads();
    return -1;
}


// ----------------------------------------------------- segment sources
// Where a consumer tile kernel takes its keys from.
enum SegMode : int {
    kSegSorted = 0,   // sorted into shared memory: sl[0 .. L)
    kSegGlobal = 1,   // key_gid[s .. s + L), already in gid order
    kSegStream = 2,   // overflowed slab: streamed in gid order from all Gaussians
};
struct Seg {
    uint32_t s, L;
    int mode;
};

// Open the tile's key segment; all threads must call.  Direct binning
// (cs.slab): every thread reads the tile's count (one broadcast load, no
// barrier on the critical path); close_segment re-zeroes it at the end of
// the kernel.  *cursor is set to 0 for kSegStream.
template <int NT = 256, int SMAX = kSortMax>
__device__ __forceinline__ Seg open_segment(const Proj* __restrict__ proj,
                                            uint32_t* __restrict__ key_gid,
                                            const uint32_t* __restrict__ tile_range,
                                            bool presorted, const ChainState& cs, int n, int T,
                                            const TileCtx& t, uint32_t* sl, uint32_t* scratch8,
                                            uint32_t* cursor) {
    const int tt = t.img * T + t.tile;
    if (cs.slab != nullptr) {
        // written by the producer kernel (visible after griddepcontrol.wait);
        // re-zeroed by thread 0 only after the CTA's last barrier
        const uint32_t count = __ldcg(&cs.tile_count[(size_t)tt * cs.cstride]);
        const uint32_t s = (uint32_t)tt * cs.slab_cap;
        if (count > cs.slab_cap) {
            if (threadIdx.x == 0) {
                *cursor = 0u;
                if (cs.seg_stats != nullptr) atomicAdd(&cs.seg_stats[0], 1u);
            }
            __syncthreads();
            return Seg{s, count, kSegStream};
        }
        if (count > (uint32_t)SMAX && threadIdx.x == 0 && cs.seg_stats != nullptr)
            atomicAdd(&cs.seg_stats[1], 1u);
        const int r = sorted_segment<NT, SMAX>(proj, key_gid, s, s + count, n, t.img, t.tx,
                                               t.ty, sl, scratch8);
        return Seg{s, count, r >= 0 ? kSegSorted : kSegGlobal};
    }
    const uint32_t s = tile_range[tt], e = tile_range[tt + 1];
    if (presorted) return Seg{s, e - s, kSegGlobal};
    const int r = sorted_segment<NT, SMAX>(proj, key_gid, s, e, n, t.img, t.tx, t.ty, sl, scratch8);
    return Seg{s, e - s, r >= 0 ? kSegSorted : kSegGlobal};
}

// Direct binning, at the end of a consumer kernel (thread 0): leave the
// tile's count zero for the next producer; CTA 0 publishes the producer's key
// total, resets the partial-slot allocator and (chained fit) advances the
// step counter.  The next kernel runs after this grid completes.
__device__ __forceinline__ void close_segment(const ChainState& cs, int tt) {
    if (threadIdx.x != 0 || cs.slab == nullptr) return;
    cs.tile_count[(size_t)tt * cs.cstride] = 0u;
    if (tt == 0) {
        if (cs.n_keys != nullptr) {
            *cs.n_keys = *cs.n_keys_acc;
            *cs.n_keys_acc = 0u;
        }
        if (cs.alloc_counter != nullptr) *cs.alloc_counter = 0u;
        if (cs.step_counter != nullptr) *cs.step_counter += 1u;
        if (cs.adam_consts != nullptr) {
            const int st = (int)*cs.step_read;
            const float lr_t = ldexpf(cs.lr0, -((st - 1) / cs.half_every));
            cs.adam_consts[0] = lr_t;
            cs.adam_consts[1] = (float)(1.0 / (1.0 - pow((double)cs.b1, (double)st)));
            cs.adam_consts[2] = (float)(1.0 / (1.0 - pow((double)cs.b2, (double)st)));
            if (cs.adan) {      // the same expressions as adan_kernel's
                cs.adam_consts[3] = (float)(1.0 / sqrt(1.0 - pow((double)cs.b3, (double)st)));
                cs.adam_consts[4] = 1.0f - lr_t * cs.wd;
                cs.adam_consts[5] = st == 1 ? 1.0f : 0.0f;
            }
        }
    }
}

// kSegStream: gather the next `want` (<= 256) Gaussians of image img whose
// tile rectangle contains (tx, ty), in gid order, from *cursor on, into
// out[0 ..).  Returns how many were found (want unless the image ran out).
// All threads must call.
template <int NT = 256>
__device__ __forceinline__ int stream_keys(const Proj* __restrict__ proj, int n, int img, int tx,
                                           int ty, int want, uint32_t* cursor, uint32_t* out,
                                           uint32_t* scratch8) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int got = 0;
    while (got < want) {
        const uint32_t cur = *cursor;
        if (cur >= (uint32_t)n) break;
        const uint32_t gi = cur + threadIdx.x;
        const bool hit = gi < (uint32_t)n && covers_tile(proj, (uint32_t)(img * n) + gi, tx, ty);
        const unsigned m = __ballot_sync(kFull, hit);
        if (lane == 0) scratch8[warp] = __popc(m);
        __syncthreads();
        int before = 0, tot = 0;
#pragma unroll
        for (int w = 0; w < NT / 32; ++w) {
            const int c = (int)scratch8[w];
            before += w < warp ? c : 0;
            tot += c;
        }
        const int take = min(tot, want - got);
        const int rank = before + __popc(m & lanemask_lt());
        if (hit && rank < take) out[got + rank] = (uint32_t)(img * n) + gi;
        __syncthreads();
        if (take == tot) {
            if (threadIdx.x == 0) *cursor = cur + blockDim.x;
        } else if (hit && rank == take - 1) {
            *cursor = gi + 1u;
        }
        got += take;
        __syncthreads();
    }
    return got;
}

// The gids of batch [base, base + 256) of the segment: thread i < returned
// count gets key base + i.  All threads must call (kSegStream gathers the
// batch block-wide into sl).
template <int NT = 256, int NB = kBatch>
__device__ __forceinline__ int batch_gid(const Seg& sg, uint32_t base, const uint32_t* key_gid,
                                         uint32_t* sl, const Proj* __restrict__ proj, int n,
                                         const TileCtx& t, uint32_t* cursor, uint32_t* scratch8,
                                         uint32_t& gid) {
    int cnt = (int)min((uint32_t)NB, sg.L - base);
    if (sg.mode == kSegStream) {
        cnt = stream_keys<NT>(proj, n, t.img, t.tx, t.ty, cnt, cursor, sl, scratch8);
        gid = (int)threadIdx.x < cnt ? sl[threadIdx.x] : 0u;
    } else if (sg.mode == kSegSorted) {
        gid = (int)threadIdx.x < cnt ? sl[base + threadIdx.x] : 0u;
    } else {
        gid = (int)threadIdx.x < cnt ? key_gid[sg.s + base + threadIdx.x] : 0u;
    }
    return cnt;
}

}  // namespace gi
