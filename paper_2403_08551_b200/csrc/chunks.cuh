// Gaussian-parallel tile passes: every staged record's in-tile box (row-major
// pixels) is cut into work-balanced chunks, one per lane, and a lane walks
// its chunk pair by pair -- every evaluated (pixel, Gaussian) pair is an
// in-box pair (no warp-culling waste, no per-warp candidate lists).  Used by
// the fused tile kernels of fused.cu for BOTH passes:
//
//   forward (Eq. 7)  C(p) = sum_n c'_n exp(-sigma_n(p)): each pair
//       adds round(c' w 2^s) to the pixel's 32-bit fixed-point accumulator in
//       shared memory (integer atomics: the sum is exact and independent of
//       the order the lanes run in, so the result is deterministic without
//       sorting the tile's keys); s is chosen per batch from the largest |c'|
//       so that no term exceeds 2^22 and no batch sum 2^30.  Per batch the
//       integer sums are converted once to fp32 and added to the pixel's fp32
//       accumulator (batch order).
//   backward (App. A): the chunk accumulates the 8 sums of
//       backward.cu's pass 2 (dc', and the five gamma-weighted moments).
//
// The planner is backward_tile_kernel's pass-2 planner generalised to NT
// lanes: C is the smallest of three candidates >= ceil(sum w / NT) whose
// chunk count fits the NT lanes (C = max w, one chunk per record, always
// fits); full chunks first, remainders in descending size so a warp's lanes
// run nearly equal trip counts.
#pragma once
#include "raster_common.cuh"

namespace gi {

// floor(a / b) for 0 <= a < 2^16, 1 <= b < 2^16 given rb ~ 1/b within 1 ulp
// (rcp.approx): (a + 1/2) / b is at least 0.5 / b away from an integer and the
// product's relative error (< 1.5 2^-23) moves it by less than that.
__device__ __forceinline__ uint32_t chunk_div(uint32_t a, float rb) {
    return (uint32_t)(((float)a + 0.5f) * rb);
}
__device__ __forceinline__ float chunk_rcp(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// Fixed-point forward accumulation: round(x 2^s) as a 32-bit integer by one
// FMA with the magic constant 1.5 2^23 (exact round-to-nearest-even for
// |x 2^s| <= 2^22), minus the constant's bits.
constexpr float kFixMagic = 12582912.0f;          // 1.5 * 2^23
constexpr int kFixMagicBits = 0x4B400000;

template <int NT>
struct ChunkShared {
    uint32_t item[NT];        // chunk: record | k0 << 8 | k1 << 17
    uint32_t jplan[NT];       // record j: fstart | nf << 9 | rpos << 18 | has_remainder << 27
    uint32_t hist[64];        // remainder-size bins -> their first item
    uint4 pa[NT / 32];        // per-warp (sum w, max w, max |c'| bits)
    uint2 pb[NT / 32];
    uint32_t pc[NT / 32];
    uint32_t n_items;
};

struct ChunkPlanOut {
    uint32_t n_items;
    float scale, inv_scale;   // 2^s, 2^-s of the fixed-point forward
};

// Plan the chunks of a staged batch of cnt <= NT records (one per thread).  Thread j < cnt brings
// its record's in-tile pair count wj and max(|c'_r|, |c'_g|, |c'_b|) (as
// float bits).  Writes ch.item[0 .. n_items) and ch.jplan[0 .. cnt); all
// threads must call; ends with a barrier.
// Planner for batches of few records (cnt <= 7/16 NT; 3 barriers): C =
// ceil(tot / (NT - cnt)), so that the chunk count sum ceil(w / C) <= tot / C
// + cnt <= NT; all full chunks first (record-major), then the remainders in
// record order, from one block scan of packed counts.  Two barriers fewer than the
// candidate search below at the price of up to NT / (NT - cnt) longer
// chunks: C2 init tile kernel 28.7 -> 27.7 us; on batches of many records
// (dense tiles) the longer chunks cost more than the barriers (fitted proxy
// 118 -> 125 us), so those keep the candidate planner.
template <int NT, bool kIlv>
__device__ __forceinline__ ChunkPlanOut plan_chunks_few(ChunkShared<NT>& ch, int cnt, uint32_t wj,
                                                        uint32_t cabs_bits) {
    constexpr int NW = NT / 32;
    const int j = threadIdx.x, lane = j & 31, warp = j >> 5;
    {
        const uint32_t ws = __reduce_add_sync(kFull, wj);
        const uint32_t cm = __reduce_max_sync(kFull, cabs_bits);
        if (lane == 0) ch.pa[warp] = make_uint4(ws, 0u, cm, 0u);
    }
    __syncthreads();
    uint32_t tot, cmx;
    {
        const uint4 x = lane < NW ? ch.pa[lane] : make_uint4(0u, 0u, 0u, 0u);
        tot = __reduce_add_sync(kFull, x.x);
        cmx = __reduce_max_sync(kFull, x.z);
    }
    const uint32_t room = max((uint32_t)NT - (uint32_t)cnt, 1u);
    const uint32_t C = max((tot + room - 1u) / room, 1u);
    // contiguous: nf chunks of C + a remainder; interleaved: ceil(wj / C)
    // chunks of ~wj / nc pairs (the same count)
    const uint32_t nf = chunk_div(wj, chunk_rcp((float)C)), rm = wj - nf * C;
    const uint32_t nc = nf + (rm != 0u ? 1u : 0u);
    // contiguous: the full chunks (all of length C) first, record-major, then
    // the remainders in record order -- one scan of (nf | has_remainder << 16)
    // gives both offsets, so the lanes of a warp mostly walk equal lengths
    const uint32_t val = kIlv ? nc : (nf | (rm != 0u ? 1u << 16 : 0u));
    uint32_t incl = val;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) ch.pc[warp] = incl;
    __syncthreads();
    uint32_t excl, Fp;
    {
        const uint32_t x = lane < NW ? ch.pc[lane] : 0u;
        Fp = __reduce_add_sync(kFull, x);
        excl = incl - val + __reduce_add_sync(kFull, lane < warp ? x : 0u);
    }
    uint32_t F;
    if constexpr (kIlv) {
        F = Fp;
        if (j < cnt) {     // chunk i of record j walks pairs i, i + nc, ...
            for (uint32_t i = 0; i < nc; ++i) ch.item[excl + i] = (uint32_t)j | i << 8 | nc << 17;
            ch.jplan[j] = excl | nc << 9;
        }
    } else {
        const uint32_t Ffull = Fp & 0xffffu;
        F = Ffull + (Fp >> 16);
        if (j < cnt) {
            const uint32_t fstart = excl & 0xffffu, rpos = Ffull + (excl >> 16);
            GI_ASSERT(fstart + nf <= (uint32_t)NT && (rm == 0u || rpos < (uint32_t)NT));
            for (uint32_t i = 0; i < nf; ++i)
                ch.item[fstart + i] = (uint32_t)j | (i * C) << 8 | ((i + 1u) * C) << 17;
            if (rm != 0u) ch.item[rpos] = (uint32_t)j | (nf * C) << 8 | wj << 17;
            ch.jplan[j] = fstart | nf << 9 | rpos << 18 | (rm != 0u ? 1u << 27 : 0u);
        }
    }
    const int e = cmx == 0u ? 0 : (int)((cmx >> 23) & 0xffu) - 126;
    const int s = min(max(22 - e, -100), 100);
    __syncthreads();
    ChunkPlanOut out;
    out.n_items = F;
    out.scale = ldexpf(1.0f, s);
    // a non-finite colour poisons the batch's pixels (as an fp32 sum would)
    out.inv_scale = cmx >= 0x7f800000u ? __int_as_float(0x7fffffff) : ldexpf(1.0f, -s);
    return out;
}

template <int NT, bool kIlv>
__device__ __forceinline__ ChunkPlanOut plan_chunks_many(ChunkShared<NT>& ch, int cnt, uint32_t wj,
                                                         uint32_t cabs_bits) {
    constexpr int NW = NT / 32;
    constexpr uint32_t kLog = NT == 256 ? 8u : (NT == 128 ? 7u : 6u);
    static_assert(NT == 256 || NT == 128 || NT == 64, "NT");
    const int j = threadIdx.x, lane = j & 31, warp = j >> 5;
    if (j < 64) ch.hist[j] = 0u;
    {   // (1) sum and max of w, max |c'| over the batch
        const uint32_t ws = __reduce_add_sync(kFull, wj), wm = __reduce_max_sync(kFull, wj);
        const uint32_t cm = __reduce_max_sync(kFull, cabs_bits);
        if (lane == 0) ch.pa[warp] = make_uint4(ws, wm, cm, 0u);
    }
    __syncthreads();
    uint32_t tot, mx, cmx;
    {
        const uint4 x = lane < NW ? ch.pa[lane] : make_uint4(0u, 0u, 0u, 0u);
        tot = __reduce_add_sync(kFull, x.x);
        mx = __reduce_max_sync(kFull, x.y);
        cmx = __reduce_max_sync(kFull, x.z);
    }
    // (2) chunk counts of the candidate chunk sizes
    const uint32_t c0 = max((tot + (uint32_t)NT - 1u) >> kLog, 1u);
    const uint32_t c1 = c0 + ((c0 + 3u) >> 2), c2 = c0 + ((c0 + 1u) >> 1);
    {
        uint32_t n01 = 0, n2 = 0;
        if (j < cnt) {
            n01 = chunk_div(wj + c0 - 1u, chunk_rcp((float)c0)) |
                  chunk_div(wj + c1 - 1u, chunk_rcp((float)c1)) << 16;
            n2 = chunk_div(wj + c2 - 1u, chunk_rcp((float)c2));
        }
        n01 = __reduce_add_sync(kFull, n01);
        n2 = __reduce_add_sync(kFull, n2);
        if (lane == 0) ch.pb[warp] = make_uint2(n01, n2);
    }
    __syncthreads();
    uint32_t C = max(mx, 1u);
    {
        const uint2 x = lane < NW ? ch.pb[lane] : make_uint2(0u, 0u);
        const uint32_t n01 = __reduce_add_sync(kFull, x.x), n2 = __reduce_add_sync(kFull, x.y);
        if (n2 <= (uint32_t)NT) C = c2;
        if ((n01 >> 16) <= (uint32_t)NT) C = c1;
        if ((n01 & 0xffffu) <= (uint32_t)NT) C = c0;
    }
    // (3) full chunks: block scan of their counts; remainders: size bins.
    // Interleaved: records of >= 2 chunks (ceil(wj / C), lengths ~wj / nc)
    // in the scanned region, one-chunk records (the whole record) binned
    uint32_t nf, rm;
    if constexpr (kIlv) {
        const uint32_t nc = chunk_div(wj + C - 1u, chunk_rcp((float)C));
        nf = nc >= 2u ? nc : 0u;
        rm = nc == 1u ? wj : 0u;
    } else {
        nf = chunk_div(wj, chunk_rcp((float)C));
        rm = wj - nf * C;
    }
    uint32_t incl = nf;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) ch.pc[warp] = incl;
    const uint32_t rbin = 64u - min(rm, 64u);        // larger remainder -> lower bin
    uint32_t rrank = 0;
    if (rm != 0u) rrank = atomicAdd(&ch.hist[rbin], 1u);
    __syncthreads();
    uint32_t F, fstart;
    {
        const uint32_t x = lane < NW ? ch.pc[lane] : 0u;
        F = __reduce_add_sync(kFull, x);
        fstart = incl - nf + __reduce_add_sync(kFull, lane < warp ? x : 0u);
    }
    if (warp == 0) {
        const uint32_t h0 = ch.hist[2 * lane], h1 = ch.hist[2 * lane + 1];
        const uint32_t v = h0 + h1;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, x, o);
            if (lane >= o) x += y;
        }
        ch.hist[2 * lane] = F + x - v;
        ch.hist[2 * lane + 1] = F + x - v + h0;
        if (lane == 31) ch.n_items = F + x;
    }
    __syncthreads();
    const uint32_t rpos = rm != 0u ? ch.hist[rbin] + rrank : 0u;
    if (j < cnt) {
        if constexpr (kIlv) {
            for (uint32_t i = 0; i < nf; ++i) ch.item[fstart + i] = (uint32_t)j | i << 8 | nf << 17;
            if (rm != 0u) ch.item[rpos] = (uint32_t)j | 1u << 17;
        } else {
            for (uint32_t i = 0; i < nf; ++i)
                ch.item[fstart + i] = (uint32_t)j | (i * C) << 8 | ((i + 1u) * C) << 17;
            if (rm != 0u) ch.item[rpos] = (uint32_t)j | (nf * C) << 8 | wj << 17;
        }
        ch.jplan[j] = fstart | nf << 9 | rpos << 18 | (rm != 0u ? 1u << 27 : 0u);
    }
    // s: the largest |c'| rounded up to a power of two, 2^e >= max |c'|; then
    // |c' w 2^s| <= 2^22 per term and a batch of <= 256 terms stays < 2^30
    const int e = cmx == 0u ? 0 : (int)((cmx >> 23) & 0xffu) - 126;
    const int s = min(max(22 - e, -100), 100);
    __syncthreads();
    ChunkPlanOut out;
    out.n_items = ch.n_items;
    out.scale = ldexpf(1.0f, s);
    // a non-finite colour poisons the batch's pixels (as an fp32 sum would)
    out.inv_scale = cmx >= 0x7f800000u ? __int_as_float(0x7fffffff) : ldexpf(1.0f, -s);
    return out;
}

// batches of <= 7/16 NT records take plan_chunks_few (3/8: render -0.8 %;
// 1/2: the fitted proxy's tile kernel 118 -> 127 us; 5/16: C2 fit -3 %)
#ifndef GI_FEW_NUM
#define GI_FEW_NUM 7
#endif
#ifndef GI_FEW_DEN
#define GI_FEW_DEN 16
#endif
// kIlv: interleaved chunks (walk_chunk_ilv) instead of contiguous ones.
template <int NT, bool kIlv = false>
__device__ __forceinline__ ChunkPlanOut plan_chunks(ChunkShared<NT>& ch, int cnt, uint32_t wj,
                                                    uint32_t cabs_bits) {
    // cnt is uniform over the CTA
    return cnt * GI_FEW_DEN <= NT * GI_FEW_NUM ? plan_chunks_few<NT, kIlv>(ch, cnt, wj, cabs_bits)
                             : plan_chunks_many<NT, kIlv>(ch, cnt, wj, cabs_bits);
}

// The pixel walk of one chunk: record r's in-tile box, row-major pairs
// [k0, k1).  Calls f(pixel index, u, v, w) per pair, with (u, v) the factored
// conic offsets (sigma log2 e = u^2 + v^2) and w = exp(-sigma).
template <class SR, typename F>
__device__ __forceinline__ void walk_chunk(const SR& sr, uint32_t it, F&& f) {
    const int r = (int)(it & 0xffu);
    const int k0 = (int)((it >> 8) & 0x1ffu), k1 = (int)(it >> 17);
    const float4 A = sr.a[r];          // {a, b, c, c'r}
    const float4 B = sr.b[r];          // {c'g, c'b, mx, my}
    const float2 O = sr.o[r];          // {u0, v0}
    const uint32_t box = sr.c[r].x;
    const int lx0 = box & 0xff, lx1 = (box >> 8) & 0xff, ly0 = (box >> 16) & 0xff;
    const int wdt = lx1 - lx0 + 1;
    const int row = (int)chunk_div((uint32_t)k0, chunk_rcp((float)wdt)), col = k0 - row * wdt;
    // row-major walk: dx steps by 1 and wraps half a pixel past the box's
    // last column (far above the stepping's rounding); c dy (+ v0) advances
    // by c per row
    const float dx0 = ((float)lx0 + 0.5f) - B.z;
    const float dx1 = ((float)lx1 + 1.0f) - B.z;
    float dx = ((float)(lx0 + col) + 0.5f) - B.z;
    float cdy = fmaf(A.z, ((float)(ly0 + row) + 0.5f) - B.w, O.y);
    int p = (ly0 + row) * kTile + lx0 + col;
    const int wrap = kTile - wdt;
    GI_ASSERT(k0 >= 0 && k0 <= k1 && k1 <= wdt * ((int)(box >> 24) - ly0 + 1));
    for (int k = k0; k < k1; ++k) {
        GI_ASSERT(p >= 0 && p < kTilePix);
        const float u = fmaf(A.x, dx, O.x);
        const float v = fmaf(A.y, dx, cdy);
        const float w = ex2_approx(fmaf(-u, u, -(v * v)));
        f(p, A, B, u, v, w);
        ++p;
        dx += 1.0f;
        if (dx > dx1) {
            p += wrap;
            dx = dx0;
            cdy += A.z;
        }
    }
}

// The interleaved walk (plan_chunks<NT, true>): record r's in-tile box,
// row-major pair index k = k0, k0 + n, k0 + 2n, ... < w (the record's n
// chunks interleave, so the lanes walking one record touch adjacent pixels at
// each step and their shared-memory accumulators fall in distinct banks).
// The render kernel uses it (C2 frame 53.6k -> 55.0k FPS); on the fit kernel
// the chunk lengths (~w / n, no longer exactly C) balance the warps worse
// than the bank conflicts cost (C2 tile kernel 28.4 -> 29.5 us).
template <class SR, typename F>
__device__ __forceinline__ void walk_chunk_ilv(const SR& sr, uint32_t it, F&& f) {
    const int r = (int)(it & 0xffu);
    const int k0 = (int)((it >> 8) & 0x1ffu), n = (int)((it >> 17) & 0x1ffu);
    const float4 A = sr.a[r];          // {a, b, c, c'r}
    const float4 B = sr.b[r];          // {c'g, c'b, mx, my}
    const float2 O = sr.o[r];          // {u0, v0}
    const uint32_t box = sr.c[r].x;
    const int lx0 = box & 0xff, lx1 = (box >> 8) & 0xff, ly0 = (box >> 16) & 0xff, ly1 = box >> 24;
    const int wdt = lx1 - lx0 + 1;
    const float rw = chunk_rcp((float)wdt);
    const int row = (int)chunk_div((uint32_t)k0, rw), col = k0 - row * wdt;
    const int srow = (int)chunk_div((uint32_t)n, rw), scol = n - srow * wdt;
    const int cnt = (int)chunk_div((uint32_t)(wdt * (ly1 - ly0 + 1) - k0 + n - 1),
                                   chunk_rcp((float)n));   // pairs of this chunk
    // dx steps by scol and wraps half a pixel past the box's last column (far
    // above the stepping's rounding); c dy (+ v0) advances by c per row
    const float dx1 = ((float)lx1 + 1.0f) - B.z;
    const float fscol = (float)scol, fwdt = (float)wdt, cstep = A.z * (float)srow;
    float dx = ((float)(lx0 + col) + 0.5f) - B.z;
    float cdy = fmaf(A.z, ((float)(ly0 + row) + 0.5f) - B.w, O.y);
    int p = (ly0 + row) * kTile + lx0 + col;
    const int pstep = srow * kTile + scol, wrap = kTile - wdt;
    for (int k = 0; k < cnt; ++k) {
        GI_ASSERT(p >= 0 && p < kTilePix);
        const float u = fmaf(A.x, dx, O.x);
        const float v = fmaf(A.y, dx, cdy);
        const float w = ex2_approx(fmaf(-u, u, -(v * v)));
        f(p, A, B, u, v, w);
        p += pstep;
        dx += fscol;
        cdy += cstep;
        if (dx > dx1) {
            p += wrap;
            dx -= fwdt;
            cdy += A.z;
        }
    }
}

}  // namespace gi
