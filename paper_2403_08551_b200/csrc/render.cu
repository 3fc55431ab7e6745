// a3. Forward accumulated summation, Eq. 7:
//     C_i = sum_{n in tile list, i in box_n} c'_n exp(-sigma_n)
// No transmittance, no depth order, no early termination: every
// covering Gaussian contributes.  Terms are summed in ascending gid (the
// tile's segment is brought into gid order in shared memory first), so the
// image is deterministic run-to-run.  FP32 + MUFU bound; see
// raster_common.cuh for the CTA layout.
#include <cstdlib>

#include "raster_common.cuh"

namespace gi {
namespace {

struct RenderShared {
    StagedRecords sr;
    WarpLists wl;
    alignas(16) uint32_t sl[kSortMax];
    uint32_t scratch[kWarps];
    uint32_t cursor;
};

#ifndef GI_RENDER_MINB
#define GI_RENDER_MINB 8
#endif
__global__ void __launch_bounds__(256, GI_RENDER_MINB) render_kernel(const Proj* __restrict__ proj,
                                                     uint32_t* __restrict__ key_gid,
                                                     const uint32_t* __restrict__ tile_range,
                                                     int n, int W, int H, int T, int TX,
                                                     bool presorted, float* __restrict__ image,
                                                     ChainState cs) {
    __shared__ RenderShared sh;
    const TileCtx t = make_tile_ctx(W, H, TX, cs.row1 > 0 ? cs.row0 : 0);
    griddep_wait();
    griddep_trigger();
    // presorted: the segment comes from gi_bin (already in gid order); else it
    // comes from direct binning and is ordered here
    const Seg sg = open_segment(proj, key_gid, tile_range, presorted, cs, n, T, t, sh.sl,
                                sh.scratch, &sh.cursor);
    float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f;
    for (uint32_t base = 0; base < sg.L; base += kBatch) {
        if (base > 0) __syncthreads();
        uint32_t gid;
        const int cnt = batch_gid(sg, base, key_gid, sh.sl, proj, n, t, &sh.cursor, sh.scratch, gid);
        if ((int)threadIdx.x < cnt) stage_gid(sh.sr, proj, gid, threadIdx.x, t);
        __syncthreads();
        const int nl = build_warp_list(sh.sr, sh.wl, cnt, t);
        forward_batch(sh.sr, sh.wl, nl, t, acc0, acc1, acc2);
    }
    if (t.in_image) {
        const size_t P = (size_t)W * H;
        float* im = image + (size_t)t.img * 3 * P + (size_t)t.y * W + t.x;
        im[0] = acc0;
        im[P] = acc1;
        im[2 * P] = acc2;
    }
    close_segment(cs, t.img * T + t.tile);
}

// ---- two pixels per thread (the default; GI_RENDER2=0 selects the
// one-pixel render_kernel above for A/B): 128 threads per tile, warp w covers
// the 8x8 block (w & 1 -> x half, w >> 1 -> y half); lane l holds the pixels
// (l & 7, l >> 3) and (l & 7, (l >> 3) + 4) of it, so a record's loads, dx
// and u serve two pixels.  Half the warps per tile: the per-warp work
// (ordering share, list building) halves, which pays on sparse tiles (C3:
// 21.2k -> 24.4k FPS) and on long segments (fitted proxy, decoded clouds);
// 8x8 culling evaluates more lane-pairs than 8x4, which evens it out at the
// C2 init scale.
// 12 CTAs per SM (40 registers; was 9 / 56): C3 frame 24.4k -> 25.7k FPS,
// 64-image frames -0.7 %
#ifndef GI_RENDER2_MINB
#define GI_RENDER2_MINB 12
#endif
constexpr int kSortMaxR2 = 1024;     // 4 KB sort buffer; longer segments are rebuilt in order
struct Render2Shared {
    StagedRecords sr;
    uint4 ent[4][kBatch];            // (record, pixel-0 lane mask, pixel-1 lane mask)
    alignas(16) uint32_t sl[kSortMaxR2];
    uint32_t scratch[kWarps];
    uint32_t cursor;
};

__global__ void __launch_bounds__(128, GI_RENDER2_MINB) render2_kernel(const Proj* __restrict__ proj,
                                                      uint32_t* __restrict__ key_gid,
                                                      const uint32_t* __restrict__ tile_range,
                                                      int n, int W, int H, int T, int TX,
                                                      bool presorted, float* __restrict__ image,
                                                      ChainState cs) {
    __shared__ Render2Shared sh;
    TileCtx t;
    t.tx = blockIdx.x;
    t.row0 = cs.row1 > 0 ? cs.row0 : 0;
    t.ty = t.row0 + blockIdx.y;
    t.img = blockIdx.z;
    t.tile = blockIdx.y * TX + t.tx;
    t.row1 = t.row0 + gridDim.y;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int lx = (warp & 1) * 8 + (lane & 7), ly = (warp >> 1) * 8 + (lane >> 3);
    const float cx = (float)lx + 0.5f, cy0 = (float)ly + 0.5f;
    const int csh = (warp & 1) * 8, rsh = (warp >> 1) * 8;
    griddep_wait();
    griddep_trigger();
    const Seg sg = open_segment<128, kSortMaxR2>(proj, key_gid, tile_range, presorted, cs, n, T,
                                                 t, sh.sl, sh.scratch, &sh.cursor);
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, b0 = 0.f, b1 = 0.f, b2 = 0.f;
    const uint32_t bit = 1u << lane;
    for (uint32_t base = 0; base < sg.L; base += kBatch) {
        if (base > 0) __syncthreads();
        uint32_t gid;
        const int cnt = batch_gid<128>(sg, base, key_gid, sh.sl, proj, n, t, &sh.cursor, sh.scratch, gid);
        if ((int)threadIdx.x < cnt) stage_gid(sh.sr, proj, gid, threadIdx.x, t);
        __syncthreads();
        // this warp's candidate list: records whose box meets its 8x8 block
        int nl = 0;
        for (int q = 0; q < cnt; q += 32) {
            const int j = q + lane;
            uint32_t m0 = 0u, m1 = 0u;
            if (j < cnt) {
                const uint32_t masks = sh.sr.c[j].y;
                const uint32_t cols = (masks >> csh) & 0xffu;
                const uint32_t rows = (masks >> (16 + rsh)) & 0xffu;
                m0 = (((rows & 0xfu) * 0x00204081u) & 0x01010101u) * cols;
                m1 = (((rows >> 4) * 0x00204081u) & 0x01010101u) * cols;
            }
            const unsigned hit = __ballot_sync(kFull, (m0 | m1) != 0u);
            if ((m0 | m1) != 0u) sh.ent[warp][nl + __popc(hit & lanemask_lt())] = make_uint4((uint32_t)j, m0, m1, 0u);
            nl += __popc(hit);
        }
        __syncwarp();
        const uint4* ent = sh.ent[warp];
#pragma unroll 2
        for (int k = 0; k < nl; ++k) {
            const uint4 en = ent[k];
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
    const size_t P = (size_t)W * H;
    const int x = t.tx * kTile + lx, y = t.ty * kTile + ly;
    if (x < W) {
        float* im = image + (size_t)t.img * 3 * P + (size_t)y * W + x;
        if (y < H) {
            im[0] = a0;
            im[P] = a1;
            im[2 * P] = a2;
        }
        if (y + 4 < H) {
            im[4 * (size_t)W] = b0;
            im[P + 4 * (size_t)W] = b1;
            im[2 * P + 4 * (size_t)W] = b2;
        }
    }
    close_segment(cs, t.img * T + t.tile);
}

bool use_render2() {
    static const bool on = [] {
        const char* e = std::getenv("GI_RENDER2");
        return e == nullptr || e[0] != '0';
    }();
    return on;
}

}  // namespace

cudaError_t launch_render(const Proj* proj, uint32_t* key_gid, const uint32_t* tile_range, int n,
                          const gi_frame& f, bool presorted, float* image, const ChainState& cs,
                          cudaStream_t s, bool decode) {
    const int TX = tiles_x(f.width);
    const int rows = cs.row1 > 0 ? cs.row1 - cs.row0 : tiles_y(f.height);   // NEXT-4 window
    const int T = TX * rows;
    if (rows <= 0) return cudaSuccess;
    if (use_render3(T * f.batch, n, T))   // Gaussian-parallel forward (fused.cu)
        return launch_fused_render(proj, key_gid, tile_range, n, f, presorted, image, cs, s, decode);
    cudaError_t e = use_render2()
        ? launch_pdl(render2_kernel, dim3(TX, rows, f.batch), dim3(128), s, proj, key_gid,
                     tile_range, n, f.width, f.height, T, TX, presorted, image, cs)
        : launch_pdl(render_kernel, dim3(TX, rows, f.batch), dim3(256), s, proj, key_gid,
                     tile_range, n, f.width, f.height, T, TX, presorted, image, cs);
    note_launches(1);
    return e;
}

}  // namespace gi
