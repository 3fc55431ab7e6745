// a3. Forward accumulated summation, Eq. 7:
//     C_i = sum_{n in tile list, i in box_n} c'_n exp(-sigma_n)
// No transmittance, no depth order, no early termination: every
// covering Gaussian contributes.  Terms are summed in ascending gid (the
// tile's segment is brought into gid order in shared memory first), so the
// image is deterministic run-to-run.  FP32 + MUFU bound; see
// raster_common.cuh for the CTA layout.
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

}  // namespace

cudaError_t launch_render(const Proj* proj, uint32_t* key_gid, const uint32_t* tile_range, int n,
                          const gi_frame& f, bool presorted, float* image, const ChainState& cs,
                          cudaStream_t s) {
    const int TX = tiles_x(f.width);
    const int rows = cs.row1 > 0 ? cs.row1 - cs.row0 : tiles_y(f.height);   // NEXT-4 window
    const int T = TX * rows;
    if (rows <= 0) return cudaSuccess;
    cudaError_t e = launch_pdl(render_kernel, dim3(TX, rows, f.batch), dim3(256), s, proj, key_gid,
                               tile_range, n, f.width, f.height, T, TX, presorted, image, cs);
    note_launches(1);
    return e;
}

}  // namespace gi
