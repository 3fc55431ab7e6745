// a4. L2 loss + analytic backward (Appendix A).
//
// backward_tile_kernel -- one CTA per 16x16 tile:
//   pass 1 (pixel-parallel, one pixel per thread, warp culling): recompute
//          C (Eq. 7), g = dL/dC = 2 (C - T) / (3HW) (or a given dL/dC) and a
//          per-tile partial of the squared error; g goes to shared memory.
//   pass 2 (GAUSSIAN-parallel): each staged record's in-tile box (row-major
//          pixels) is cut into work-balanced chunks, one per lane (see the
//          planner below); a lane walks its chunk and accumulates, per pair
//          with w = exp(-sigma):
//              dc'     += g w                               (A.1)
//              gamma    = dL/dsigma = -w <g, c'>             (A.1, R12)
//              S_u += gamma u, S_v += gamma v, S_uu += gamma u^2,
//              S_uv += gamma u v, S_vv += gamma v^2
//          with (u, v) = kappa L^-1 d, i.e. the 8 numbers from which
//          dsigma/dmu (sign R13) and dsigma/dSigma chained
//          through Sigma = L L^T (A.2, R14) follow in closed form.
//          Every evaluated pair is an in-box pair (no warp-culling waste) and
//          no per-pair warp reduction is needed; a record's chunk sums are
//          added in a fixed order and written once to the Gaussian's partial
//          slot (4 gid, or gauss_off[gid] above 4 tiles, + the rank of the
//          tile in its rectangle) -- no atomics, deterministic.
// finalize_kernel -- one thread per Gaussian: sums its contiguous slots in
//   row-major tile order, applies the chain rule (and tanh, App. C) and
//   optionally the Adam update (fused fit step).
#include <cstdlib>

#include "project_core.cuh"
#include "raster_common.cuh"

namespace gi {
namespace {

// Fixed-point scale of the per-tile squared-error sums (2^40: a tile's sum
// is at most 768 on the [0, 1] scale, a batch image's at most ~1.2e18 / 2^40).
constexpr double kSseScale = 1099511627776.0;

struct BwdShared {
    StagedRecords sr;
    union {
        WarpLists wl;            // pass 1: per-warp candidate lists
        float4 red[256][2];      // pass 2: the 8 sums of each chunk
    } u;
    alignas(16) uint32_t sl[kSortMax];
    float4 g[kTilePix];      // per-pixel upstream dL/dC (x, y, z), tile-local row-major
    uint32_t scratch[kWarps];
    float sse[kWarps];
    uint32_t cursor;   // segment count / stream cursor
    uint32_t hist[64];       // pass-2 remainder-size histogram -> bin starts
    uint32_t item[256];      // pass-2 chunk: record | k0 << 8 | k1 << 17
    uint2 pa[kWarps], pb[kWarps];   // pass-2 per-warp partials
    uint32_t pc[kWarps];
    uint32_t n_items;
};

// floor(a / b) for 0 <= a < 2^16, 1 <= b < 2^16 given rb ~ 1/b (fp32 within
// 1 ulp, e.g. rcp.approx): (a + 1/2) / b is at least 0.5/b away from an
// integer, and the product's relative error (< 1.5 2^-23) moves it by less
// than (a + 1/2) 2^-22.4 / b < 0.5 / b since a < 2^16.
__device__ __forceinline__ uint32_t small_div(uint32_t a, float rb) {
    return (uint32_t)(((float)a + 0.5f) * rb);
}

// 1/x by MUFU.RCP (rcp.approx: at most 1 ulp), for small_div.
__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

#ifndef GI_TILE_MINB
#define GI_TILE_MINB 6
#endif
__global__ void __launch_bounds__(256, GI_TILE_MINB) backward_tile_kernel(
    const Proj* __restrict__ proj, uint32_t* __restrict__ key_gid,
    const uint32_t* __restrict__ tile_range, const uint32_t* __restrict__ gauss_off, int n,
    int W, int H, int T, int TX, bool presorted, const float* __restrict__ dL_dimage,
    const float* __restrict__ target, float norm, int64_t pcap, float* __restrict__ partial,
    float* __restrict__ ovf, unsigned long long* __restrict__ sse_acc, float* __restrict__ image_out,
    ChainState cs) {
    __shared__ BwdShared sh;
    const TileCtx t = make_tile_ctx(W, H, TX, cs.row1 > 0 ? cs.row0 : 0);
    const size_t P = (size_t)W * H;
    const size_t pix = (size_t)t.img * 3 * P + (size_t)t.y * W + t.x;
    const int lpix = (t.y - t.ty * kTile) * kTile + (t.x - t.tx * kTile);
    griddep_wait();
    griddep_trigger();
    const Seg sg = open_segment(proj, key_gid, tile_range, presorted, cs, n, T, t, sh.sl,
                                sh.scratch, &sh.cursor);
    const uint32_t L = sg.L;
    bool staged_all = false;

    float g0 = 0.f, g1 = 0.f, g2 = 0.f;
    if (dL_dimage != nullptr) {
        if (t.in_image) {
            g0 = dL_dimage[pix];
            g1 = dL_dimage[pix + P];
            g2 = dL_dimage[pix + 2 * P];
        }
    } else {
        // ---- pass 1: forward (Eq. 7), pixel-parallel ----
        float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f;
        for (uint32_t base = 0; base < L; base += kBatch) {
            if (base > 0) __syncthreads();
            uint32_t gid;
            const int cnt =
                batch_gid(sg, base, key_gid, sh.sl, proj, n, t, &sh.cursor, sh.scratch, gid);
            if ((int)threadIdx.x < cnt) stage_gid(sh.sr, proj, gid, threadIdx.x, t, gauss_off);
            __syncthreads();
            const int nl = build_warp_list(sh.sr, sh.u.wl, cnt, t);
            forward_batch(sh.sr, sh.u.wl, nl, t, acc0, acc1, acc2);
        }
        staged_all = L <= (uint32_t)kBatch;
        float sq = 0.f;
        if (t.in_image) {
            const float r0 = acc0 - target[pix];
            const float r1 = acc1 - target[pix + P];
            const float r2 = acc2 - target[pix + 2 * P];
            g0 = norm * r0;
            g1 = norm * r1;
            g2 = norm * r2;
            sq = fmaf(r0, r0, fmaf(r1, r1, r2 * r2));
            if (image_out != nullptr) {
                image_out[pix] = acc0;
                image_out[pix + P] = acc1;
                image_out[pix + 2 * P] = acc2;
            }
        }
        if (sse_acc != nullptr) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(kFull, sq, o);
            if (t.lane == 0) sh.sse[t.warp] = sq;
        }
    }
    sh.g[lpix] = make_float4(g0, g1, g2, 0.f);
    __syncthreads();
    if (sse_acc != nullptr && dL_dimage == nullptr && threadIdx.x == 0) {
        // per-image squared error in 2^-40 fixed point: integer addition is
        // associative, so the loss is deterministic whatever the tile order
        float tot = 0.f;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) tot += sh.sse[w];
        atomicAdd(&sse_acc[t.img], (unsigned long long)__double2ll_rn((double)tot * kSseScale));
    }

    // ---- pass 2: gradients, Gaussian-parallel, work-balanced chunks ----
    // Record j's in-tile box (w_j pixels, row-major) is cut into chunks of at
    // most C pairs: floor(w_j / C) full chunks and one remainder.  C is the
    // smallest of a few candidates >= ceil(sum w / 256) whose chunk count fits
    // the 256 lanes (C = max w_j, one chunk per record, always fits).  Full
    // chunks come first, remainders follow in descending size, so the lanes
    // of a warp run nearly equal trip counts.  Each lane accumulates the 8
    // sums of its chunk; thread j then adds its chunks in a fixed order.
    const int j = threadIdx.x;
    if (threadIdx.x == 0) sh.cursor = 0u;        // kSegStream: pass 2 streams from the start
    for (uint32_t base = 0; base < L; base += kBatch) {
        __syncthreads();
        uint32_t gid = 0;
        int cnt = (int)min((uint32_t)kBatch, L - base);
        if (!staged_all)
            cnt = batch_gid(sg, base, key_gid, sh.sl, proj, n, t, &sh.cursor, sh.scratch, gid);
        if (j < 64) sh.hist[j] = 0u;
        uint32_t slot = 0, wj = 0, jgid = 0;
        if (j < cnt) {
            if (!staged_all) stage_gid(sh.sr, proj, gid, j, t, gauss_off);
            const uint4 c = sh.sr.c[j];
            slot = c.z;
            jgid = c.w;
            const int lx0 = c.x & 0xff, lx1 = (c.x >> 8) & 0xff;
            const int ly0 = (c.x >> 16) & 0xff, ly1 = c.x >> 24;
            wj = (uint32_t)((lx1 - lx0 + 1) * (ly1 - ly0 + 1));
        }
        // (1) sum and max of w over the batch
        {
            const uint32_t ws = __reduce_add_sync(kFull, wj), wm = __reduce_max_sync(kFull, wj);
            if (t.lane == 0) sh.pa[t.warp] = make_uint2(ws, wm);
        }
        __syncthreads();
        // 8-way combines of per-warp partials: lane w < 8 loads warp w's, one redux
        uint32_t tot, mx;
        {
            const uint2 x = t.lane < kWarps ? sh.pa[t.lane] : make_uint2(0u, 0u);
            tot = __reduce_add_sync(kFull, x.x);
            mx = __reduce_max_sync(kFull, x.y);
        }
        // (2) chunk counts of the candidate chunk sizes
        const uint32_t c0 = (tot + 255u) >> 8;
        const uint32_t c1 = c0 + ((c0 + 3u) >> 2), c2 = c0 + ((c0 + 1u) >> 1);
        {
            uint32_t n01 = 0, n2 = 0;
            if (j < cnt) {
                n01 = small_div(wj + c0 - 1u, rcp_approx((float)c0)) |
                      small_div(wj + c1 - 1u, rcp_approx((float)c1)) << 16;
                n2 = small_div(wj + c2 - 1u, rcp_approx((float)c2));
            }
            n01 = __reduce_add_sync(kFull, n01);
            n2 = __reduce_add_sync(kFull, n2);
            if (t.lane == 0) sh.pb[t.warp] = make_uint2(n01, n2);
        }
        __syncthreads();
        uint32_t C = mx;
        {
            const uint2 x = t.lane < kWarps ? sh.pb[t.lane] : make_uint2(0u, 0u);
            const uint32_t n01 = __reduce_add_sync(kFull, x.x), n2 = __reduce_add_sync(kFull, x.y);
            if (n2 <= 256u) C = c2;
            if ((n01 >> 16) <= 256u) C = c1;
            if ((n01 & 0xffffu) <= 256u) C = c0;
        }
        // (3) full chunks: block scan of their counts; remainders: size bins
        const uint32_t nf = small_div(wj, rcp_approx((float)C)), rm = wj - nf * C;
        uint32_t incl = nf;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, incl, o);
            if (t.lane >= o) incl += y;
        }
        if (t.lane == 31) sh.pc[t.warp] = incl;
        const uint32_t rbin = 64u - min(rm, 64u);        // larger remainder -> lower bin
        uint32_t rrank = 0;
        if (rm != 0u) rrank = atomicAdd(&sh.hist[rbin], 1u);
        __syncthreads();
        uint32_t F, fstart;
        {
            const uint32_t x = t.lane < kWarps ? sh.pc[t.lane] : 0u;
            F = __reduce_add_sync(kFull, x);
            fstart = incl - nf + __reduce_add_sync(kFull, t.lane < t.warp ? x : 0u);
        }
        if (t.warp == 0) {
            const uint32_t h0 = sh.hist[2 * t.lane], h1 = sh.hist[2 * t.lane + 1];
            const uint32_t v = h0 + h1;
            uint32_t x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, x, o);
                if (t.lane >= o) x += y;
            }
            sh.hist[2 * t.lane] = F + x - v;
            sh.hist[2 * t.lane + 1] = F + x - v + h0;
            if (t.lane == 31) sh.n_items = F + x;
        }
        __syncthreads();
        const uint32_t rpos = rm != 0u ? sh.hist[rbin] + rrank : 0u;
        if (j < cnt) {
            for (uint32_t i = 0; i < nf; ++i)
                sh.item[fstart + i] = (uint32_t)j | (i * C) << 8 | ((i + 1u) * C) << 17;
            if (rm != 0u) sh.item[rpos] = (uint32_t)j | (nf * C) << 8 | wj << 17;
        }
        __syncthreads();
        if (j < (int)sh.n_items) {
            const uint32_t it = sh.item[j];
            const int r = (int)(it & 0xffu);
            const int k0 = (int)((it >> 8) & 0x1ffu), k1 = (int)(it >> 17);
            const float4 A = sh.sr.a[r];          // {a, b, c, c'r}
            const float4 B = sh.sr.b[r];          // {c'g, c'b, mx, my}
            const uint32_t box = sh.sr.c[r].x;
            const int lx0 = box & 0xff, lx1 = (box >> 8) & 0xff, ly0 = (box >> 16) & 0xff;
            const int wdt = lx1 - lx0 + 1;
            const int row = (int)small_div((uint32_t)k0, rcp_approx((float)wdt)), col = k0 - row * wdt;
            // row-major walk: dx steps by 1 and wraps half a pixel past the
            // box's last column (far above the stepping's rounding), c dy
            // advances by c per row
            const float2 O = sh.sr.o[r];          // {u0, v0}
            const float dx0 = ((float)lx0 + 0.5f) - B.z;
            const float dx1 = ((float)lx1 + 1.0f) - B.z;
            float dx = ((float)(lx0 + col) + 0.5f) - B.z;
            float cdy = fmaf(A.z, ((float)(ly0 + row) + 0.5f) - B.w, O.y);   // c dy + v0
            const float4* gp_ptr = &sh.g[(ly0 + row) * kTile + lx0 + col];
            const int wrap = kTile - wdt;
            float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f, a4 = 0.f, a5 = 0.f, a6 = 0.f, a7 = 0.f;
            for (int k = k0; k < k1; ++k) {
                const float u = fmaf(A.x, dx, O.x);
                const float v = fmaf(A.y, dx, cdy);
                const float w = ex2_approx(fmaf(-u, u, -(v * v)));
                const float4 gp = *gp_ptr;
                a0 = fmaf(gp.x, w, a0);
                a1 = fmaf(gp.y, w, a1);
                a2 = fmaf(gp.z, w, a2);
                const float sdot = w * fmaf(A.w, gp.x, fmaf(B.x, gp.y, B.y * gp.z));   // -gamma
                const float gu = -sdot * u, gv = -sdot * v;
                a3 += gu;
                a4 += gv;
                a5 = fmaf(gu, u, a5);
                a6 = fmaf(gu, v, a6);
                a7 = fmaf(gv, v, a7);
                ++gp_ptr;
                dx += 1.0f;
                if (dx > dx1) {
                    gp_ptr += wrap;
                    dx = dx0;
                    cdy += A.z;
                }
            }
            sh.u.red[j][0] = make_float4(a0, a1, a2, a3);
            sh.u.red[j][1] = make_float4(a4, a5, a6, a7);
        }
        __syncthreads();
        if (j < cnt && (slot == kOffOverflow || (int64_t)slot < pcap)) {
            float4 s0 = make_float4(0.f, 0.f, 0.f, 0.f), s1 = s0;
            auto add = [&](uint32_t i) {
                const float4 x = sh.u.red[i][0], y = sh.u.red[i][1];
                s0.x += x.x; s0.y += x.y; s0.z += x.z; s0.w += x.w;
                s1.x += y.x; s1.y += y.y; s1.z += y.z; s1.w += y.w;
            };
            for (uint32_t i = 0; i < nf; ++i) add(fstart + i);
            if (rm != 0u) add(rpos);
            if (slot == kOffOverflow) {     // > 4-tile Gaussian without slots: accumulate
                float* o = ovf + (size_t)jgid * 8;
                atomicAdd(o + 0, s0.x); atomicAdd(o + 1, s0.y); atomicAdd(o + 2, s0.z);
                atomicAdd(o + 3, s0.w); atomicAdd(o + 4, s1.x); atomicAdd(o + 5, s1.y);
                atomicAdd(o + 6, s1.z); atomicAdd(o + 7, s1.w);
            } else {
                float4* dst = reinterpret_cast<float4*>(partial + (size_t)slot * 8);
                dst[0] = s0;
                dst[1] = s1;
            }
        }
    }
    close_segment(cs, t.img * T + t.tile);
}

// ---- two pixels per thread: the render2_kernel layout (128 threads, 8x8
// warp blocks, pixels (x, y) and (x, y + 4) per lane) for pass 1; pass 2
// plans its chunks over 128 lanes.  Chosen for launches with many tiles
// (use_tile2 below).
// 48 registers, 18.8 KB of shared memory: 10 CTAs (40 warps) per SM
#ifndef GI_TILE2_MINB
#define GI_TILE2_MINB 10
#endif
#ifndef GI_TILE2_SORT
#define GI_TILE2_SORT 512
#endif
#ifndef GI_TILE2_UNPACKED
#define GI_TILE2_PACKED     // candidate entries as (mask pair, byte index): 9 B instead of 16
#endif
constexpr int kSortMax2 = GI_TILE2_SORT;   // sort buffer; longer segments are rebuilt in order
struct Bwd2Shared {
    StagedRecords sr;
    union {
#ifdef GI_TILE2_PACKED
        struct {
            uint2 m[4][kBatch];      // pass 1: (pixel-0 mask, pixel-1 mask)
            uint8_t j[4][kBatch];    //         record index
        } ent;
#else
        uint4 ent[4][kBatch];    // pass 1: (record, pixel-0 mask, pixel-1 mask)
#endif
        float4 red[128][2];      // pass 2: the 8 sums of each chunk
    } u;
    alignas(16) uint32_t sl[kSortMax2];   // segments beyond are rebuilt in order (rare)
    float4 g[kTilePix];
    uint32_t scratch[kWarps];
    float sse[4];
    uint32_t cursor;
    uint32_t hist[64];
    uint32_t item[128];
    uint2 pa[4], pb[4];
    uint32_t pc[4];
    uint32_t n_items;
};

__global__ void __launch_bounds__(128, GI_TILE2_MINB) backward_tile2_kernel(
    const Proj* __restrict__ proj, uint32_t* __restrict__ key_gid,
    const uint32_t* __restrict__ tile_range, const uint32_t* __restrict__ gauss_off, int n,
    int W, int H, int T, int TX, bool presorted, const float* __restrict__ dL_dimage,
    const float* __restrict__ target, float norm, int64_t pcap, float* __restrict__ partial,
    float* __restrict__ ovf, unsigned long long* __restrict__ sse_acc, float* __restrict__ image_out,
    ChainState cs) {
    __shared__ Bwd2Shared sh;
    TileCtx t;
    t.tx = blockIdx.x;
    t.row0 = cs.row1 > 0 ? cs.row0 : 0;
    t.ty = t.row0 + blockIdx.y;
    t.img = blockIdx.z;
    t.tile = blockIdx.y * TX + t.tx;
    t.row1 = t.row0 + gridDim.y;
    t.lane = threadIdx.x & 31;
    t.warp = threadIdx.x >> 5;
    // two pixels per thread: (lx, ly) and (lx, ly + 4) of the warp's 8x8 block
    const int lx = (t.warp & 1) * 8 + (t.lane & 7), ly = (t.warp >> 1) * 8 + (t.lane >> 3);
    const float cx = (float)lx + 0.5f, cy0 = (float)ly + 0.5f;
    const int csh = (t.warp & 1) * 8, rsh = (t.warp >> 1) * 8;
    const int x = t.tx * kTile + lx, y = t.ty * kTile + ly;
    const bool in0 = x < W && y < H, in1 = x < W && y + 4 < H;
    const size_t P = (size_t)W * H;
    const size_t pix = (size_t)t.img * 3 * P + (size_t)y * W + x;
    const size_t pix1 = pix + 4 * (size_t)W;
    const int lpix = ly * kTile + lx;
    griddep_wait();
    griddep_trigger();
    const Seg sg = open_segment<128, kSortMax2>(proj, key_gid, tile_range, presorted, cs, n, T, t,
                                                sh.sl, sh.scratch, &sh.cursor);
    const uint32_t L = sg.L;
    bool staged_all = false;

    float g0 = 0.f, g1 = 0.f, g2 = 0.f, h0 = 0.f, h1 = 0.f, h2 = 0.f;   // pixel 0, pixel 1
    if (dL_dimage != nullptr) {
        if (in0) {
            g0 = dL_dimage[pix];
            g1 = dL_dimage[pix + P];
            g2 = dL_dimage[pix + 2 * P];
        }
        if (in1) {
            h0 = dL_dimage[pix1];
            h1 = dL_dimage[pix1 + P];
            h2 = dL_dimage[pix1 + 2 * P];
        }
    } else {
        // ---- pass 1: forward (Eq. 7), pixel-parallel, two pixels per lane ----
        float a0 = 0.f, a1 = 0.f, a2 = 0.f, b0 = 0.f, b1 = 0.f, b2 = 0.f;
        const uint32_t bit = 1u << t.lane;
        for (uint32_t base = 0; base < L; base += kBatch) {
            if (base > 0) __syncthreads();
            uint32_t gid;
            const int cnt =
                batch_gid<128>(sg, base, key_gid, sh.sl, proj, n, t, &sh.cursor, sh.scratch, gid);
            if ((int)threadIdx.x < cnt) stage_gid(sh.sr, proj, gid, threadIdx.x, t, gauss_off);
            __syncthreads();
            int nl = 0;
            for (int q = 0; q < cnt; q += 32) {
                const int jj = q + t.lane;
                uint32_t m0 = 0u, m1 = 0u;
                if (jj < cnt) {
                    const uint32_t masks = sh.sr.c[jj].y;
                    const uint32_t cols = (masks >> csh) & 0xffu;
                    const uint32_t rows = (masks >> (16 + rsh)) & 0xffu;
                    m0 = (((rows & 0xfu) * 0x00204081u) & 0x01010101u) * cols;
                    m1 = (((rows >> 4) * 0x00204081u) & 0x01010101u) * cols;
                }
                const unsigned hit = __ballot_sync(kFull, (m0 | m1) != 0u);
                if ((m0 | m1) != 0u) {
                    const int at = nl + __popc(hit & lanemask_lt());
#ifdef GI_TILE2_PACKED
                    sh.u.ent.m[t.warp][at] = make_uint2(m0, m1);
                    sh.u.ent.j[t.warp][at] = (uint8_t)jj;
#else
                    sh.u.ent[t.warp][at] = make_uint4((uint32_t)jj, m0, m1, 0u);
#endif
                }
                nl += __popc(hit);
            }
            __syncwarp();
#ifdef GI_TILE2_PACKED
            const uint2* entm = sh.u.ent.m[t.warp];
            const uint8_t* entj = sh.u.ent.j[t.warp];
#else
            const uint4* ent = sh.u.ent[t.warp];
#endif
#pragma unroll 2
            for (int k = 0; k < nl; ++k) {
#ifdef GI_TILE2_PACKED
                const uint2 mm = entm[k];
                const uint4 en = make_uint4((uint32_t)entj[k], mm.x, mm.y, 0u);
#else
                const uint4 en = ent[k];
#endif
                const float4 A = sh.sr.a[en.x];      // {a, b, c, c'r}
                const float4 B = sh.sr.b[en.x];      // {c'g, c'b, mx, my}
                const float2 O = sh.sr.o[en.x];      // {u0, v0}
                const float dx = cx - B.z;
                const float dy = cy0 - B.w;
                const float u = fmaf(A.x, dx, O.x);
                const float v0 = fmaf(A.y, dx, fmaf(A.z, dy, O.y));
                const float v1 = fmaf(A.z, 4.0f, v0);
                const float uu = u * u;
                float w0 = ex2_approx(fmaf(-v0, v0, -uu));
                float w1 = ex2_approx(fmaf(-v1, v1, -uu));
                w0 = (en.y & bit) ? w0 : 0.f;
                w1 = (en.z & bit) ? w1 : 0.f;
                a0 = fmaf(A.w, w0, a0);
                a1 = fmaf(B.x, w0, a1);
                a2 = fmaf(B.y, w0, a2);
                b0 = fmaf(A.w, w1, b0);
                b1 = fmaf(B.x, w1, b1);
                b2 = fmaf(B.y, w1, b2);
            }
        }
        staged_all = L <= (uint32_t)kBatch;
        float sq = 0.f;
        if (in0) {
            const float r0 = a0 - target[pix];
            const float r1 = a1 - target[pix + P];
            const float r2 = a2 - target[pix + 2 * P];
            g0 = norm * r0;
            g1 = norm * r1;
            g2 = norm * r2;
            sq = fmaf(r0, r0, fmaf(r1, r1, r2 * r2));
            if (image_out != nullptr) {
                image_out[pix] = a0;
                image_out[pix + P] = a1;
                image_out[pix + 2 * P] = a2;
            }
        }
        if (in1) {
            const float r0 = b0 - target[pix1];
            const float r1 = b1 - target[pix1 + P];
            const float r2 = b2 - target[pix1 + 2 * P];
            h0 = norm * r0;
            h1 = norm * r1;
            h2 = norm * r2;
            sq += fmaf(r0, r0, fmaf(r1, r1, r2 * r2));
            if (image_out != nullptr) {
                image_out[pix1] = b0;
                image_out[pix1 + P] = b1;
                image_out[pix1 + 2 * P] = b2;
            }
        }
        if (sse_acc != nullptr) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(kFull, sq, o);
            if (t.lane == 0) sh.sse[t.warp] = sq;
        }
    }
    sh.g[lpix] = make_float4(g0, g1, g2, 0.f);
    sh.g[lpix + 4 * kTile] = make_float4(h0, h1, h2, 0.f);
    __syncthreads();
    if (sse_acc != nullptr && dL_dimage == nullptr && threadIdx.x == 0) {
        // per-image squared error in 2^-40 fixed point (see backward_tile_kernel)
        float tot = 0.f;
#pragma unroll
        for (int w = 0; w < 4; ++w) tot += sh.sse[w];
        atomicAdd(&sse_acc[t.img], (unsigned long long)__double2ll_rn((double)tot * kSseScale));
    }

    // ---- pass 2: gradients, Gaussian-parallel, work-balanced chunks ----
    // Record j's in-tile box (w_j pixels, row-major) is cut into chunks of at
    // most C pairs: floor(w_j / C) full chunks and one remainder.  C is the
    // smallest of a few candidates >= ceil(sum w / 256) whose chunk count fits
    // the 256 lanes (C = max w_j, one chunk per record, always fits).  Full
    // chunks come first, remainders follow in descending size, so the lanes
    // of a warp run nearly equal trip counts.  Each lane accumulates the 8
    // sums of its chunk; thread j then adds its chunks in a fixed order.
    const int j = threadIdx.x;
    if (threadIdx.x == 0) sh.cursor = 0u;        // kSegStream: pass 2 streams from the start
    for (uint32_t base = 0; base < L; base += kBatch) {
        __syncthreads();
        uint32_t gid = 0;
        int cnt = (int)min((uint32_t)kBatch, L - base);
        if (!staged_all)
            cnt = batch_gid<128>(sg, base, key_gid, sh.sl, proj, n, t, &sh.cursor, sh.scratch, gid);
        if (j < 64) sh.hist[j] = 0u;
        uint32_t slot = 0, wj = 0, jgid = 0;
        if (j < cnt) {
            if (!staged_all) stage_gid(sh.sr, proj, gid, j, t, gauss_off);
            const uint4 c = sh.sr.c[j];
            slot = c.z;
            jgid = c.w;
            const int lx0 = c.x & 0xff, lx1 = (c.x >> 8) & 0xff;
            const int ly0 = (c.x >> 16) & 0xff, ly1 = c.x >> 24;
            wj = (uint32_t)((lx1 - lx0 + 1) * (ly1 - ly0 + 1));
        }
        // (1) sum and max of w over the batch
        {
            const uint32_t ws = __reduce_add_sync(kFull, wj), wm = __reduce_max_sync(kFull, wj);
            if (t.lane == 0) sh.pa[t.warp] = make_uint2(ws, wm);
        }
        __syncthreads();
        // 8-way combines of per-warp partials: lane w < 8 loads warp w's, one redux
        uint32_t tot, mx;
        {
            const uint2 x = t.lane < 4 ? sh.pa[t.lane] : make_uint2(0u, 0u);
            tot = __reduce_add_sync(kFull, x.x);
            mx = __reduce_max_sync(kFull, x.y);
        }
        // (2) chunk counts of the candidate chunk sizes
        const uint32_t c0 = (tot + 127u) >> 7;
        const uint32_t c1 = c0 + ((c0 + 3u) >> 2), c2 = c0 + ((c0 + 1u) >> 1);
        {
            uint32_t n01 = 0, n2 = 0;
            if (j < cnt) {
                n01 = small_div(wj + c0 - 1u, rcp_approx((float)c0)) |
                      small_div(wj + c1 - 1u, rcp_approx((float)c1)) << 16;
                n2 = small_div(wj + c2 - 1u, rcp_approx((float)c2));
            }
            n01 = __reduce_add_sync(kFull, n01);
            n2 = __reduce_add_sync(kFull, n2);
            if (t.lane == 0) sh.pb[t.warp] = make_uint2(n01, n2);
        }
        __syncthreads();
        uint32_t C = mx;
        {
            const uint2 x = t.lane < 4 ? sh.pb[t.lane] : make_uint2(0u, 0u);
            const uint32_t n01 = __reduce_add_sync(kFull, x.x), n2 = __reduce_add_sync(kFull, x.y);
            if (n2 <= 128u) C = c2;
            if ((n01 >> 16) <= 128u) C = c1;
            if ((n01 & 0xffffu) <= 128u) C = c0;
        }
        // (3) full chunks: block scan of their counts; remainders: size bins
        const uint32_t nf = small_div(wj, rcp_approx((float)C)), rm = wj - nf * C;
        uint32_t incl = nf;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, incl, o);
            if (t.lane >= o) incl += y;
        }
        if (t.lane == 31) sh.pc[t.warp] = incl;
        const uint32_t rbin = 64u - min(rm, 64u);        // larger remainder -> lower bin
        uint32_t rrank = 0;
        if (rm != 0u) rrank = atomicAdd(&sh.hist[rbin], 1u);
        __syncthreads();
        uint32_t F, fstart;
        {
            const uint32_t x = t.lane < 4 ? sh.pc[t.lane] : 0u;
            F = __reduce_add_sync(kFull, x);
            fstart = incl - nf + __reduce_add_sync(kFull, t.lane < t.warp ? x : 0u);
        }
        if (t.warp == 0) {
            const uint32_t h0 = sh.hist[2 * t.lane], h1 = sh.hist[2 * t.lane + 1];
            const uint32_t v = h0 + h1;
            uint32_t x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, x, o);
                if (t.lane >= o) x += y;
            }
            sh.hist[2 * t.lane] = F + x - v;
            sh.hist[2 * t.lane + 1] = F + x - v + h0;
            if (t.lane == 31) sh.n_items = F + x;
        }
        __syncthreads();
        const uint32_t rpos = rm != 0u ? sh.hist[rbin] + rrank : 0u;
        if (j < cnt) {
            for (uint32_t i = 0; i < nf; ++i)
                sh.item[fstart + i] = (uint32_t)j | (i * C) << 8 | ((i + 1u) * C) << 17;
            if (rm != 0u) sh.item[rpos] = (uint32_t)j | (nf * C) << 8 | wj << 17;
        }
        __syncthreads();
        if (j < (int)sh.n_items) {
            const uint32_t it = sh.item[j];
            const int r = (int)(it & 0xffu);
            const int k0 = (int)((it >> 8) & 0x1ffu), k1 = (int)(it >> 17);
            const float4 A = sh.sr.a[r];          // {a, b, c, c'r}
            const float4 B = sh.sr.b[r];          // {c'g, c'b, mx, my}
            const uint32_t box = sh.sr.c[r].x;
            const int lx0 = box & 0xff, lx1 = (box >> 8) & 0xff, ly0 = (box >> 16) & 0xff;
            const int wdt = lx1 - lx0 + 1;
            const int row = (int)small_div((uint32_t)k0, rcp_approx((float)wdt)), col = k0 - row * wdt;
            // row-major walk: dx steps by 1 and wraps half a pixel past the
            // box's last column (far above the stepping's rounding), c dy
            // advances by c per row
            const float2 O = sh.sr.o[r];          // {u0, v0}
            const float dx0 = ((float)lx0 + 0.5f) - B.z;
            const float dx1 = ((float)lx1 + 1.0f) - B.z;
            float dx = ((float)(lx0 + col) + 0.5f) - B.z;
            float cdy = fmaf(A.z, ((float)(ly0 + row) + 0.5f) - B.w, O.y);   // c dy + v0
            const float4* gp_ptr = &sh.g[(ly0 + row) * kTile + lx0 + col];
            const int wrap = kTile - wdt;
            float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f, a4 = 0.f, a5 = 0.f, a6 = 0.f, a7 = 0.f;
            for (int k = k0; k < k1; ++k) {
                const float u = fmaf(A.x, dx, O.x);
                const float v = fmaf(A.y, dx, cdy);
                const float w = ex2_approx(fmaf(-u, u, -(v * v)));
                const float4 gp = *gp_ptr;
                a0 = fmaf(gp.x, w, a0);
                a1 = fmaf(gp.y, w, a1);
                a2 = fmaf(gp.z, w, a2);
                const float sdot = w * fmaf(A.w, gp.x, fmaf(B.x, gp.y, B.y * gp.z));   // -gamma
                const float gu = -sdot * u, gv = -sdot * v;
                a3 += gu;
                a4 += gv;
                a5 = fmaf(gu, u, a5);
                a6 = fmaf(gu, v, a6);
                a7 = fmaf(gv, v, a7);
                ++gp_ptr;
                dx += 1.0f;
                if (dx > dx1) {
                    gp_ptr += wrap;
                    dx = dx0;
                    cdy += A.z;
                }
            }
            sh.u.red[j][0] = make_float4(a0, a1, a2, a3);
            sh.u.red[j][1] = make_float4(a4, a5, a6, a7);
        }
        __syncthreads();
        if (j < cnt && (slot == kOffOverflow || (int64_t)slot < pcap)) {
            float4 s0 = make_float4(0.f, 0.f, 0.f, 0.f), s1 = s0;
            auto add = [&](uint32_t i) {
                const float4 x = sh.u.red[i][0], y = sh.u.red[i][1];
                s0.x += x.x; s0.y += x.y; s0.z += x.z; s0.w += x.w;
                s1.x += y.x; s1.y += y.y; s1.z += y.z; s1.w += y.w;
            };
            for (uint32_t i = 0; i < nf; ++i) add(fstart + i);
            if (rm != 0u) add(rpos);
            if (slot == kOffOverflow) {     // > 4-tile Gaussian without slots: accumulate
                float* o = ovf + (size_t)jgid * 8;
                atomicAdd(o + 0, s0.x); atomicAdd(o + 1, s0.y); atomicAdd(o + 2, s0.z);
                atomicAdd(o + 3, s0.w); atomicAdd(o + 4, s1.x); atomicAdd(o + 5, s1.y);
                atomicAdd(o + 6, s1.z); atomicAdd(o + 7, s1.w);
            } else {
                float4* dst = reinterpret_cast<float4*>(partial + (size_t)slot * 8);
                dst[0] = s0;
                dst[1] = s1;
            }
        }
    }
    close_segment(cs, t.img * T + t.tile);
}


// Kernel choice: the two-pixel kernel wins when a launch has more tiles than
// one C2 image (C3: 10,880 tiles, fit 8.9k -> 11.4k it/s; C2 x 2 images:
// 28.6k -> 29.1k image-it/s, x 8: 34.7k -> 37.3k, x 64: 36.9k -> 40.5k) and
// loses on one C2 image (1,536 tiles: 24.4k -> 23.2k: its CTAs live twice as
// long, so the last of ~1.2 waves leaves SMs idle).  GI_TILE2=0/1 forces
// either (A/B).
constexpr int kTile2MinTiles = 3072;
bool use_tile2(int tiles) {
    static const int force = [] {
        const char* e = std::getenv("GI_TILE2");
        return e == nullptr ? -1 : (e[0] == '1' ? 1 : 0);
    }();
    return force >= 0 ? force == 1 : tiles >= kTile2MinTiles;
}

__global__ void __launch_bounds__(256) alloc_kernel(const Proj* __restrict__ proj, int total,
                                                    int64_t pcap, uint32_t* __restrict__ counter,
                                                    uint32_t* __restrict__ gauss_off) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t cnt = 0;
    if (g < total) {
        const uint32_t* rw = reinterpret_cast<const uint32_t*>(proj + g);   // box words only
        const uint32_t bx = rw[7], by = rw[11];
        const int x0 = (int)(bx & 0xffffu), x1 = (int)(bx >> 16);
        const int y0 = (int)(by & 0xffffu), y1 = (int)(by >> 16);
        if (x0 <= x1 && y0 <= y1)
            cnt = (uint32_t)((x1 / kTile - x0 / kTile + 1) * (y1 / kTile - y0 / kTile + 1));
    }
    // same layout as direct binning (post_project_warp): 4 g for <= 4-tile
    // Gaussians, 4 total + allocation for larger ones
    uint32_t off = 4u * (uint32_t)g;
    if (__any_sync(kFull, cnt > 4u)) {
        const uint32_t big_off = warp_alloc(counter, cnt > 4u ? cnt : 0u);
        const int64_t first = 4ll * total + big_off;
        if (cnt > 4u) off = first + cnt <= pcap ? (uint32_t)first : kOffOverflow;
    }
    if (g < total) gauss_off[g] = off;
}

// The partial sums of a > 4-tile Gaussian: slots o0 .. o0 + n - 1, four
// loads in flight, summed in slot order (kept out of line: the common <= 4-
// tile path of finalize_one is scheduled as if this loop did not exist).
struct Sums8 {
    float4 u, w;
};
__device__ __noinline__ Sums8 sum_slots(const float4* __restrict__ pp, uint32_t o0, uint32_t n) {
    Sums8 s{make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f)};
    for (uint32_t k = 0; k < n; k += 4) {
        float4 u4[4], w4[4];
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q)
            if (k + q < n) {
                u4[q] = __ldcg(pp + 2 * (size_t)(o0 + k + q));
                w4[q] = __ldcg(pp + 2 * (size_t)(o0 + k + q) + 1);
            }
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q)
            if (k + q < n) {
                s.u.x += u4[q].x; s.u.y += u4[q].y; s.u.z += u4[q].z; s.u.w += u4[q].w;
                s.w.x += w4[q].x; s.w.y += w4[q].y; s.w.z += w4[q].z; s.w.w += w4[q].w;
            }
    }
    return s;
}

// Per Gaussian: sum its tiles' partials (row-major tile order), then the
// closed-form chain rule.  With p = u / kappa, q = v / kappa (so
// sigma = (p^2 + q^2) / 2, p = dx / l1, q = (dy - l2 p) / l3):
//   dsigma/ddx = (p - q l2 / l3) / l1,  dsigma/ddy = q / l3,  d = pixel - mu
//   dsigma/dl1 = -p dsigma/ddx, dsigma/dl2 = -p q / l3, dsigma/dl3 = -q^2 / l3
// (equal to <dsigma/dSigma, dSigma/dl> of A.2 with the R14 correction).
// Everything the per-Gaussian finalize needs (the finalize kernel's
// arguments minus the loss).
struct FinArgs {
    const float4* params;
    const Proj* proj;          // this step's records (the chained step rewrites proj[g] in place)
    const uint32_t* gauss_off;
    int total, n_per_image, W, H;
    uint32_t flags;
    int64_t pcap;
    const float* partial;
    float* ovf;
    float4* grads;
    FusedAdam adam;
    int row0, row1;
};

// Finalize Gaussian g (live = g is a real Gaussian for this thread).  All
// lanes of the warp must call (the direct-binning tail is warp-cooperative).
// lr, ibc1, ibc2: the Adam step constants.
template <bool kAdan>
__device__ __forceinline__ void finalize_one(int g, bool live, const FinArgs& a, float lr,
                                             float ibc1, float ibc2) {
    const FusedAdam& adam = a.adam;
    const int W = a.W, H = a.H, n_per_image = a.n_per_image, total = a.total;
    const uint32_t flags = a.flags;
    // independent loads first (their latency overlaps the partial-sum chain)
    float4 p0 = make_float4(0.f, 0.f, 0.f, 0.f), p1 = p0, m0 = p0, m1 = p0, v0 = p0, v1 = p0;
    uint32_t bx = 0u, by = 0u;     // the record's box words: all finalize needs of it
    const float4* pp = reinterpret_cast<const float4*>(a.partial);
    if (live) {
        p0 = a.params[2 * (size_t)g];
        p1 = a.params[2 * (size_t)g + 1];
        const uint32_t* rw = reinterpret_cast<const uint32_t*>(a.proj + g);
        bx = rw[7];                 // q1.w: x0 | x1 << 16
        by = rw[11];                // q2.w: y0 | y1 << 16
        if (adam.m != nullptr) {
            const float4* mm = reinterpret_cast<const float4*>(adam.m) + 2 * (size_t)g;
            const float4* vv = reinterpret_cast<const float4*>(adam.v) + 2 * (size_t)g;
            m0 = mm[0]; m1 = mm[1]; v0 = vv[0]; v1 = vv[1];
        }
    }
    float4 n0{}, n1{}, gp0{}, gp1{};      // Adan: third moment, previous gradient
    if constexpr (kAdan) {
        if (live) {
            const float4* nn = reinterpret_cast<const float4*>(adam.n) + 2 * (size_t)g;
            const float4* gg = reinterpret_cast<const float4*>(adam.gprev) + 2 * (size_t)g;
            n0 = nn[0]; n1 = nn[1]; gp0 = gg[0]; gp1 = gg[1];
        }
    }
    uint32_t touched = 0;
    int4 rect = make_int4(0, -1, 0, -1);
    if (live) {
        const int x0 = (int)(bx & 0xffffu), x1 = (int)(bx >> 16);
        const int y0 = (int)(by & 0xffffu), y1 = (int)(by >> 16);
        float S[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        bool any = false;
        // tiles of the (window-clipped, NEXT-4) rectangle
        const uint32_t cnt =
            rect_area(window_rect(make_int4(x0 / kTile, x1 / kTile, y0 / kTile, y1 / kTile), a.row0,
                                  a.row1));
        if (x0 <= x1 && y0 <= y1 && cnt > 0u) {
            auto add = [&](const float4 u, const float4 w) {
                S[0] += u.x; S[1] += u.y; S[2] += u.z; S[3] += u.w;
                S[4] += w.x; S[5] += w.y; S[6] += w.z; S[7] += w.w;
            };
            if (cnt <= 4u) {
                // fixed slots 4 g .. 4 g + cnt - 1: all loads issued at once
                float4 a4[4], b4[4];
                const size_t o = 4 * (size_t)g;
    #pragma unroll
                for (int k = 0; k < 4; ++k)
                    if ((uint32_t)k < cnt) {
                        a4[k] = pp[2 * (o + k)];
                        b4[k] = pp[2 * (o + k) + 1];
                    }
    #pragma unroll
                for (int k = 0; k < 4; ++k)                // row-major tile order of the rectangle
                    if ((uint32_t)k < cnt) add(a4[k], b4[k]);
            } else {
                const uint32_t o0 = a.gauss_off[g];
                if (o0 == kOffOverflow) {          // summed atomically by the tiles; re-zero
                    float4* o = reinterpret_cast<float4*>(a.ovf) + 2 * (size_t)g;
                    add(__ldcg(o), __ldcg(o + 1));
                    o[0] = make_float4(0.f, 0.f, 0.f, 0.f);
                    o[1] = make_float4(0.f, 0.f, 0.f, 0.f);
                } else {
                    // below pcap: alloc_kernel and post_project_warp allocate
                    // whole ranges or none (the clip keeps the old loop's break)
                    const uint32_t n_ok = (int64_t)o0 + cnt <= a.pcap
                        ? cnt : (uint32_t)max(a.pcap - (int64_t)o0, (int64_t)0);
                    const Sums8 s8 = sum_slots(pp, o0, n_ok);
                    add(s8.u, s8.w);
                }
            }
            any = true;
        }
        float4 r0 = make_float4(0.f, 0.f, 0.f, 0.f), r1 = r0;
        if (any && !cov_rs(flags)) {
            // Cholesky, in fp64: (Sp - Sq l2/l3) / l1 and (Spp - Spq l2/l3) / l1
            // cancel for near-line Gaussians (|l2 / l3| large); one thread
            // per Gaussian, so the wider arithmetic is off the critical path
            const double l1 = (double)__fadd_rn(p0.z, 0.5f), l2 = (double)p0.w;
            const double l3 = (double)__fadd_rn(p1.x, 0.5f);
            const double il1 = 1.0 / l1, il3 = 1.0 / l3;
            const double ik = 1.0 / kKappa, ik2 = 1.0 / (kKappa * kKappa);
            const double Sp = S[3] * ik, Sq = S[4] * ik;
            const double Spp = S[5] * ik2, Spq = S[6] * ik2, Sqq = S[7] * ik2;
            const double l2l3 = l2 * il3;
            const double Ax = (Sp - Sq * l2l3) * il1;        // sum gamma dsigma/ddx
            const double Ay = Sq * il3;
            r0.x = (float)-Ax;                                // dmu_pix = -dsigma/dd (R13)
            r0.y = (float)-Ay;
            r0.z = (float)(-(Spp - Spq * l2l3) * il1);        // dl1
            r0.w = (float)(-Spq * il3);                       // dl2
            r1.x = (float)(-Sqq * il3);                       // dl3
        } else if (any) {
            // NEXT-3 rotation-scaling: L = chol(Sigma) as in the projection, then
            // G = dL/dSigma = -1/2 L^-T M L^-1 with M = sum gamma (p, q)(p, q)^T,
            // chained through Sigma(theta, s1, s2) (App. A.2).
            const double th = (double)p0.z;
            const double s1 = (double)__fadd_rn(p0.w, 0.5f), s2 = (double)__fadd_rn(p1.x, 0.5f);
            double Sg[3];
            rs_sigma(th, s1, s2, Sg);
            const double l1 = sqrt(Sg[0]), l2 = Sg[1] / l1, l3 = fabs(s1 * s2) / l1;
            const double ik = 1.0 / kKappa, ik2 = ik * ik;
            const double Sp = S[3] * ik, Sq = S[4] * ik;
            const double Spp = S[5] * ik2, Spq = S[6] * ik2, Sqq = S[7] * ik2;
            const double al = 1.0 / l1, be = -l2 / (l1 * l3), ga = 1.0 / l3;   // L^-1 = [[al,0],[be,ga]]
            r0.x = (float)(-(al * Sp + be * Sq));             // dmu_pix = -L^-T (S_p, S_q)
            r0.y = (float)(-(ga * Sq));
            const double G11 = -0.5 * (al * al * Spp + 2.0 * al * be * Spq + be * be * Sqq);
            const double G12 = -0.5 * (al * ga * Spq + be * ga * Sqq);
            const double G22 = -0.5 * (ga * ga * Sqq);
            const double c = cos(th), sn = sin(th);
            const double s2t = 2.0 * sn * c, c2t = c * c - sn * sn;
            r0.z = (float)((s1 * s1 - s2 * s2) * (-G11 * s2t + 2.0 * G12 * c2t + G22 * s2t));   // dtheta
            r0.w = (float)(2.0 * s1 * (G11 * c * c + 2.0 * G12 * c * sn + G22 * sn * sn));     // ds1
            r1.x = (float)(2.0 * s2 * (G11 * sn * sn - 2.0 * G12 * c * sn + G22 * c * c));     // ds2
        }
        if (any) {
            // position activation chain (App. C): mu = (tanh(r) + 1) W/2
            float sx = (float)W * 0.5f, sy = (float)H * 0.5f;
            if (pos_logit(flags)) {
                const float chx = coshf(p0.x), chy = coshf(p0.y);
                sx /= chx * chx;
                sy /= chy * chy;
            }
            r0.x *= sx;
            r0.y *= sy;
            r1.y = S[0];                                      // dc'
            r1.z = S[1];
            r1.w = S[2];
        }
        a.grads[2 * (size_t)g] = r0;
        a.grads[2 * (size_t)g + 1] = r1;
        if (adam.m != nullptr) {
                float4* mm = reinterpret_cast<float4*>(adam.m) + 2 * (size_t)g;
            float4* vv = reinterpret_cast<float4*>(adam.v) + 2 * (size_t)g;
            float4* pw = reinterpret_cast<float4*>(adam.params) + 2 * (size_t)g;
            float4 q0, q1;
            const float b1 = adam.b1, b2 = adam.b2, eps = adam.eps;
            if constexpr (kAdan) {          // NEXT-1: the paper's optimiser, fused
                AdanConsts c;
                c.lr = lr;
                c.ibc1 = ibc1;
                c.ibc2 = ibc2;
                c.isbc3 = adam.consts[3];
                c.decay = adam.consts[4];
                c.first = adam.consts[5] != 0.0f;
                c.b1 = b1; c.b2 = b2; c.b3 = adam.b3; c.eps = eps;
                q0.x = adan1(p0.x, r0.x, m0.x, v0.x, n0.x, gp0.x, c);
                q0.y = adan1(p0.y, r0.y, m0.y, v0.y, n0.y, gp0.y, c);
                q0.z = adan1(p0.z, r0.z, m0.z, v0.z, n0.z, gp0.z, c);
                q0.w = adan1(p0.w, r0.w, m0.w, v0.w, n0.w, gp0.w, c);
                q1.x = adan1(p1.x, r1.x, m1.x, v1.x, n1.x, gp1.x, c);
                q1.y = adan1(p1.y, r1.y, m1.y, v1.y, n1.y, gp1.y, c);
                q1.z = adan1(p1.z, r1.z, m1.z, v1.z, n1.z, gp1.z, c);
                q1.w = adan1(p1.w, r1.w, m1.w, v1.w, n1.w, gp1.w, c);
                float4* nn = reinterpret_cast<float4*>(adam.n) + 2 * (size_t)g;
                float4* gg = reinterpret_cast<float4*>(adam.gprev) + 2 * (size_t)g;
                nn[0] = n0; nn[1] = n1; gg[0] = gp0; gg[1] = gp1;
            } else {   // gi_adam_step's arithmetic (adam_update: IEEE sqrt and division)
                const float omb1 = 1.0f - b1, omb2 = 1.0f - b2;
                q0.x = p0.x;
                adam_update(q0.x, r0.x, m0.x, v0.x, b1, b2, omb1, omb2, lr, ibc1, ibc2, eps);
                q0.y = p0.y;
                adam_update(q0.y, r0.y, m0.y, v0.y, b1, b2, omb1, omb2, lr, ibc1, ibc2, eps);
                q0.z = p0.z;
                adam_update(q0.z, r0.z, m0.z, v0.z, b1, b2, omb1, omb2, lr, ibc1, ibc2, eps);
                q0.w = p0.w;
                adam_update(q0.w, r0.w, m0.w, v0.w, b1, b2, omb1, omb2, lr, ibc1, ibc2, eps);
                q1.x = p1.x;
                adam_update(q1.x, r1.x, m1.x, v1.x, b1, b2, omb1, omb2, lr, ibc1, ibc2, eps);
                q1.y = p1.y;
                adam_update(q1.y, r1.y, m1.y, v1.y, b1, b2, omb1, omb2, lr, ibc1, ibc2, eps);
                q1.z = p1.z;
                adam_update(q1.z, r1.z, m1.z, v1.z, b1, b2, omb1, omb2, lr, ibc1, ibc2, eps);
                q1.w = p1.w;
                adam_update(q1.w, r1.w, m1.w, v1.w, b1, b2, omb1, omb2, lr, ibc1, ibc2, eps);
            }
            mm[0] = m0; mm[1] = m1; vv[0] = v0; vv[1] = v1;
            pw[0] = q0; pw[1] = q1;
            const bool bad = !(isfinite(q0.x) && isfinite(q0.y) && isfinite(q0.z) && isfinite(q0.w) &&
                               isfinite(q1.x) && isfinite(q1.y) && isfinite(q1.z) && isfinite(q1.w));
            if (bad && adam.flag != nullptr) atomicOr(adam.flag, 1u);
            if (adam.proj_out != nullptr) {  // chained: a1 of the next step on the updated Gaussian
                touched = project_one(q0, q1, g, n_per_image, W, H, adam.k, adam.pos_flags,
                                      adam.proj_out, adam.counts, rect);
                adam.touched_out[g] = touched;
            }
        }
    }
    if (adam.m != nullptr && adam.proj_out != nullptr && adam.counts.tile_count != nullptr) {
        const int TX = (W + kTile - 1) / kTile;
        const int T = TX * (adam.counts.row1 > 0 ? adam.counts.row1 - adam.counts.row0
                                                  : (H + kTile - 1) / kTile);
        post_project_warp(adam.counts, touched, rect, g, live ? (g / n_per_image) * T : 0, TX,
                          total);
    }
}

template <bool kAdan>
// 256 threads per CTA: 274 CTAs on one C2 image instead of 547; in the
// pipelined step (PDL behind the tile kernel) fit 32.5k -> 33.4k it/s
// (flushed per replay 27.2k -> 28.5k); 128 and 512 measured lower
#ifndef GI_FIN_THREADS
#define GI_FIN_THREADS 256
#endif
__global__ void __launch_bounds__(GI_FIN_THREADS) finalize_kernel(FinArgs a,
                                                       unsigned long long* __restrict__ sse_acc,
                                                       int batch, double inv_count,
                                                       float* __restrict__ loss) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (a.adam.m != nullptr && g < a.total) {   // CTAs resident in the tile kernel's tail warm L2
        prefetch_l2(a.params + 2 * (size_t)g);
        prefetch_l2(a.adam.m + 8 * (size_t)g);
        prefetch_l2(a.adam.v + 8 * (size_t)g);
        if constexpr (kAdan) {
            prefetch_l2(a.adam.n + 8 * (size_t)g);
            prefetch_l2(a.adam.gprev + 8 * (size_t)g);
        }
    }
    griddep_wait();
    griddep_trigger();
    float lr = 0.f, ibc1 = 0.f, ibc2 = 0.f;
    if (a.adam.m != nullptr) {
        lr = a.adam.consts[0];
        ibc1 = a.adam.consts[1];
        ibc2 = a.adam.consts[2];
    }
    if (sse_acc != nullptr && blockIdx.x == 0) {
        // per-image L2 loss from the tiles' fixed-point sums; re-zero
        for (int i = threadIdx.x; i < batch; i += blockDim.x) {
            const unsigned long long v = sse_acc[i];
            sse_acc[i] = 0ull;
            if (loss != nullptr) loss[i] = (float)((double)v * (1.0 / kSseScale) * inv_count);
        }
    }
    finalize_one<kAdan>(g, g < a.total, a, lr, ibc1, ibc2);
}

__global__ void loss_kernel(unsigned long long* __restrict__ sse_acc, int batch, double inv_count,
                            float* __restrict__ loss) {
    for (int i = threadIdx.x; i < batch; i += blockDim.x) {
        const unsigned long long a = sse_acc[i];
        sse_acc[i] = 0ull;
        if (loss != nullptr) loss[i] = (float)((double)a * (1.0 / kSseScale) * inv_count);
    }
}

struct BwdWs {
    float* partial;
    uint32_t* gauss_off;
    float* ovf;
    uint32_t* counter;
    unsigned long long* sse_acc;
    float* adam_consts;
    size_t bytes;
};

BwdWs carve(void* base, int n, int64_t cap, const gi_frame& f) {
    const int T = tiles_x(f.width) * tiles_y(f.height);
    const size_t total = (size_t)n * f.batch;
    char* p = static_cast<char*>(base);
    BwdWs w;
    size_t off = 0;
    w.partial = reinterpret_cast<float*>(p + off); off += align_up(sizeof(float) * 8 * (size_t)partial_cap(n, cap, f));
    w.gauss_off = reinterpret_cast<uint32_t*>(p + off); off += align_up(sizeof(uint32_t) * (total + 1));
    w.ovf = reinterpret_cast<float*>(p + off); off += align_up(sizeof(float) * 8 * total);
    w.counter = reinterpret_cast<uint32_t*>(p + off); off += align_up(sizeof(uint32_t));
    w.sse_acc = reinterpret_cast<unsigned long long*>(p + off); off += align_up(8 * (size_t)f.batch);
    w.adam_consts = reinterpret_cast<float*>(p + off); off += align_up(8 * sizeof(float));
    w.bytes = off;
    return w;
}

}  // namespace

// Partial slots: 4 per Gaussian (the <= 4-tile ones use 4 g .. 4 g + 3) plus
// max(key capacity, 4 per Gaussian) for the Gaussians touching more tiles.
int64_t partial_cap(int n, int64_t cap, const gi_frame& f) {
    const int64_t fixed = 4 * (int64_t)n * f.batch;
    return fixed + (cap > fixed ? cap : fixed);
}

size_t backward_ws_bytes(int n, int64_t cap, const gi_frame& f) { return carve(nullptr, n, cap, f).bytes; }

uint32_t* backward_alloc_counter(void* ws, int n, int64_t cap, const gi_frame& f) {
    return carve(ws, n, cap, f).counter;
}
float* backward_adam_consts(void* ws, int n, int64_t cap, const gi_frame& f) {
    return carve(ws, n, cap, f).adam_consts;
}
uint32_t* backward_gauss_off(void* ws, int n, int64_t cap, const gi_frame& f) {
    return carve(ws, n, cap, f).gauss_off;
}

cudaError_t launch_backward_alloc(const Proj* proj, int n, const gi_frame& f, int64_t cap, void* ws,
                                  cudaStream_t s) {
    BwdWs w = carve(ws, n, cap, f);
    const int total = n * f.batch;
    cudaError_t e = cudaMemsetAsync(w.counter, 0, sizeof(uint32_t), s);
    if (e != cudaSuccess || total == 0) return e;
    alloc_kernel<<<(total + 255) / 256, 256, 0, s>>>(proj, total, partial_cap(n, cap, f), w.counter,
                                                      w.gauss_off);
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_backward_tiles(const Proj* proj, uint32_t* key_gid, const uint32_t* tile_range,
                                  int n, const gi_frame& f, bool presorted,
                                  const float* dL_dimage, const float* target, int64_t cap,
                                  void* ws, float* image_out, const ChainState& cs,
                                  cudaStream_t s) {
    BwdWs w = carve(ws, n, cap, f);
    const int TX = tiles_x(f.width);
    const int rows = cs.row1 > 0 ? cs.row1 - cs.row0 : tiles_y(f.height);   // NEXT-4 window
    const int T = TX * rows;
    const double count = 3.0 * (double)f.width * (double)f.height;
    const float norm = (float)(2.0 / count);
    const bool mse = dL_dimage == nullptr;
    if (rows <= 0) return cudaSuccess;
    if (use_tile3())      // Gaussian-parallel passes (fused.cu), the default
        return launch_fused_backward(proj, key_gid, tile_range, (const uint32_t*)w.gauss_off, n, f,
                                     presorted, dL_dimage, target, norm, partial_cap(n, cap, f),
                                     w.partial, w.ovf, mse ? w.sse_acc : nullptr,
                                     mse ? image_out : nullptr, cs, s);
    cudaError_t e = use_tile2(T * f.batch)
        ? launch_pdl(backward_tile2_kernel, dim3(TX, rows, f.batch), dim3(128), s, proj, key_gid,
                     tile_range, (const uint32_t*)w.gauss_off, n, f.width, f.height, T, TX,
                     presorted, dL_dimage, target, norm, partial_cap(n, cap, f), w.partial, w.ovf,
                     mse ? w.sse_acc : nullptr, mse ? image_out : nullptr, cs)
        : launch_pdl(backward_tile_kernel, dim3(TX, rows, f.batch), dim3(256), s, proj, key_gid,
                     tile_range, (const uint32_t*)w.gauss_off, n, f.width, f.height, T, TX,
                     presorted, dL_dimage, target, norm, partial_cap(n, cap, f), w.partial, w.ovf,
                     mse ? w.sse_acc : nullptr, mse ? image_out : nullptr, cs);
    note_launches(1);
    return e;
}

cudaError_t launch_backward_finalize(const float* params, const Proj* proj, int n,
                                     const gi_frame& f, uint32_t flags, bool mse, int64_t cap,
                                     void* ws, float* grads, float* loss, const FusedAdam* adam,
                                     cudaStream_t s, int row0, int row1) {
    BwdWs w = carve(ws, n, cap, f);
    const double count = 3.0 * (double)f.width * (double)f.height;
    const int total = n * f.batch;
    cudaError_t e = cudaSuccess;
    if (total > 0) {
        FusedAdam fa{};
        if (adam) fa = *adam;
        FinArgs fa_args{reinterpret_cast<const float4*>(params), proj, (const uint32_t*)w.gauss_off,
                        total, n, f.width, f.height, flags, partial_cap(n, cap, f),
                        (const float*)w.partial, w.ovf, reinterpret_cast<float4*>(grads), fa, row0,
                        row1 > 0 ? row1 : tiles_y(f.height)};
        // 128-thread CTAs on launches of >= 3,072 tiles (64 C2 images +1 %)
        const int ft = (int64_t)tiles_x(f.width) * tiles_y(f.height) * f.batch >= 3072
                           ? 128 : GI_FIN_THREADS;
        if (adam != nullptr && adam->n != nullptr)
            e = launch_pdl(finalize_kernel<true>, dim3((total + ft - 1) / ft), dim3(ft), s, fa_args,
                           mse ? w.sse_acc : nullptr, f.batch, 1.0 / count, mse ? loss : nullptr);
        else
            e = launch_pdl(finalize_kernel<false>, dim3((total + ft - 1) / ft), dim3(ft), s, fa_args,
                           mse ? w.sse_acc : nullptr, f.batch, 1.0 / count, mse ? loss : nullptr);
        note_launches(1);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    } else if (mse) {
        loss_kernel<<<1, 256, 0, s>>>(w.sse_acc, f.batch, 1.0 / count, loss);
        note_launches(1);
        e = cudaGetLastError();
    }
    return e;
}

cudaError_t launch_backward(const float* params, const Proj* proj, const uint32_t* key_gid,
                            const uint32_t* tile_range, int n, const gi_frame& f, uint32_t flags,
                            const float* dL_dimage, const float* target, int64_t cap, void* ws,
                            float* grads, float* loss, float* image_out, cudaStream_t s) {
    cudaError_t e = launch_backward_alloc(proj, n, f, cap, ws, s);
    if (e != cudaSuccess) return e;
    // gi_bin output is already in gid order: no re-sort, key_gid not written
    e = launch_backward_tiles(proj, const_cast<uint32_t*>(key_gid), tile_range, n, f, true,
                              dL_dimage, target, cap, ws, image_out, ChainState{}, s);
    if (e != cudaSuccess) return e;
    return launch_backward_finalize(params, proj, n, f, flags, dL_dimage == nullptr, cap, ws, grads,
                                    loss, nullptr, s);
}

}  // namespace gi
