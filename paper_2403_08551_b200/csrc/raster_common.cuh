// Tile rasteriser building blocks shared by the forward (render.cu) and the
// fused forward + L2 + backward (backward.cu) kernels.
//
// CTA = one 16x16 tile of one image, 256 threads, one pixel per thread.
// Warp w covers an 8x4 pixel block (w & 1 -> x half, w >> 1 -> y quarter), so
// a warp can skip a Gaussian whose box misses its block (warp culling): at
// the paper's init scale this evaluates ~3x fewer pairs than whole-tile
// evaluation.
//
// Per batch of up to 256 keys of the tile, each thread stages one record in
// shared memory, converted to TILE-LOCAL coordinates:
//   rA = {mx, my, a, b}   centre minus the tile origin, fp32 (ix - tx0 is an
//                         exact small integer, + fx rounds once)
//   rB = {c, c'r, c'g, c'b}
//   rC = {x0, x1 - x0, y0, y1 - y0}   integer box, global pixels
// so that a pair costs dx = (lx + 1/2) - mx (one FADD, no int->float
// conversion) and an unsigned range test per axis.
#pragma once
#include "gi_internal.cuh"

namespace gi {

struct TileCtx {
    int img, tile, tx, ty;        // tile coordinates
    int lane, warp;
    int x, y;                     // global pixel of this thread
    float cx, cy;                 // tile-local pixel centre (x + 1/2 - 16 tx)
    int wx0, wy0;                 // warp block origin (global pixels)
    bool in_image;
};

__device__ __forceinline__ TileCtx make_tile_ctx(int W, int H, int TX) {
    TileCtx c;
    c.tile = blockIdx.x;
    c.img = blockIdx.y;
    c.tx = c.tile % TX;
    c.ty = c.tile / TX;
    c.lane = threadIdx.x & 31;
    c.warp = threadIdx.x >> 5;
    const int lx = (c.warp & 1) * 8 + (c.lane & 7);
    const int ly = (c.warp >> 1) * 4 + (c.lane >> 3);
    c.x = c.tx * kTile + lx;
    c.y = c.ty * kTile + ly;
    c.cx = (float)lx + 0.5f;
    c.cy = (float)ly + 0.5f;
    c.wx0 = c.tx * kTile + (c.warp & 1) * 8;
    c.wy0 = c.ty * kTile + (c.warp >> 1) * 4;
    c.in_image = c.x < W && c.y < H;
    return c;
}

struct StagedRecords {
    float4 a[256];
    float4 b[256];
    int4 c[256];
};

// Stage key j = threadIdx.x of [base, base + cnt) into shared memory.
__device__ __forceinline__ void stage_record(StagedRecords& sr, const Proj* __restrict__ proj,
                                             const uint32_t* __restrict__ key_gid, uint32_t base,
                                             int cnt, const TileCtx& t, uint32_t* gid_out) {
    const int j = threadIdx.x;
    if (j < cnt) {
        const uint32_t gid = key_gid[base + j];
        const Proj r = proj[gid];
        const int ix = __float_as_int(r.q0.x), iy = __float_as_int(r.q0.y);
        const float mx = __fadd_rn((float)(ix - t.tx * kTile), r.q0.z);
        const float my = __fadd_rn((float)(iy - t.ty * kTile), r.q0.w);
        const uint32_t bx = __float_as_uint(r.q1.w), by = __float_as_uint(r.q2.w);
        const int x0 = (int)(bx & 0xffffu), x1 = (int)(bx >> 16);
        const int y0 = (int)(by & 0xffffu), y1 = (int)(by >> 16);
        sr.a[j] = make_float4(mx, my, r.q1.x, r.q1.y);
        sr.b[j] = make_float4(r.q1.z, r.q2.x, r.q2.y, r.q2.z);
        sr.c[j] = make_int4(x0, x1 - x0, y0, y1 - y0);
        if (gid_out) *gid_out = gid;
    }
}

// Does staged record j's box overlap this warp's 8x4 block?
__device__ __forceinline__ bool warp_overlaps(const int4 b, const TileCtx& t) {
    return (b.x <= t.wx0 + 7) && (b.x + b.y >= t.wx0) && (b.z <= t.wy0 + 3) && (b.z + b.w >= t.wy0);
}

__device__ __forceinline__ bool pixel_in_box(const int4 b, const TileCtx& t) {
    return ((unsigned)(t.x - b.x) <= (unsigned)b.y) & ((unsigned)(t.y - b.z) <= (unsigned)b.w);
}

// exp(-sigma) for the staged record (factored conic, MUFU.EX2), and the
// scaled offsets u = a dx, v = b dx + c dy (sigma log2 e = u^2 + v^2).
struct PairEval {
    float w, u, v;
};

__device__ __forceinline__ PairEval eval_pair(const float4 A, const float4 B, const TileCtx& t) {
    PairEval e;
    const float dx = t.cx - A.x;
    const float dy = t.cy - A.y;
    e.u = A.z * dx;
    e.v = fmaf(A.w, dx, B.x * dy);
    e.w = ex2_approx(fmaf(-e.u, e.u, -(e.v * e.v)));
    return e;
}

}  // namespace gi
