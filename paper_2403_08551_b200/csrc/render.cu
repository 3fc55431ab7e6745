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
};

__global__ void __launch_bounds__(256) render_kernel(const Proj* __restrict__ proj,
                                                     uint32_t* __restrict__ key_gid,
                                                     const uint32_t* __restrict__ tile_range,
                                                     int n, int W, int H, int T, int TX,
                                                     bool presorted, float* __restrict__ image,
                                                     ChainState cs) {
    __shared__ RenderShared sh;
    const TileCtx t = make_tile_ctx(W, H, TX);
    griddep_wait();
    griddep_trigger();
    if (threadIdx.x == 0 && cs.tile_count != nullptr) {   // leave the counters zero for the next call
        const int tt = t.img * T + t.tile;
        cs.tile_count[(size_t)tt * kCountStride] = 0u;
        cs.big_count[tt] = 0u;
        cs.fill[tt] = 0u;
        if (tt == 0 && cs.alloc_counter != nullptr) *cs.alloc_counter = 0u;
    }
    const uint32_t s = tile_range[t.img * T + t.tile];
    const uint32_t e = tile_range[t.img * T + t.tile + 1];
    // presorted: the segment comes from gi_bin (already in gid order); else it
    // comes from the fused scatter and is ordered here
    const int sorted = presorted ? -1
                                 : sorted_segment(proj, key_gid, s, e, n, t.img, t.tx, t.ty, sh.sl,
                                                  sh.scratch);
    float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f;
    for (uint32_t base = 0; base < e - s; base += 256) {
        const int cnt = (int)min(256u, e - s - base);
        if (base > 0) __syncthreads();
        if ((int)threadIdx.x < cnt) {
            const uint32_t gid = sorted >= 0 ? sh.sl[base + threadIdx.x] : key_gid[s + base + threadIdx.x];
            stage_gid(sh.sr, proj, gid, threadIdx.x, t);
        }
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
}

}  // namespace

cudaError_t launch_render(const Proj* proj, uint32_t* key_gid, const uint32_t* tile_range, int n,
                          const gi_frame& f, bool presorted, float* image, const ChainState& cs,
                          cudaStream_t s) {
    const int TX = tiles_x(f.width), T = TX * tiles_y(f.height);
    cudaError_t e = launch_pdl(render_kernel, dim3(TX, T / TX, f.batch), dim3(256), s, proj, key_gid,
                               tile_range, n, f.width, f.height, T, TX, presorted, image, cs);
    note_launches(1);
    return e;
}

}  // namespace gi
