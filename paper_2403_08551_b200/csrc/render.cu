// a3. Forward accumulated summation, Eq. 7:
//     C_i = sum_{n in tile list, i in box_n} c'_n exp(-sigma_n)
// No transmittance, no depth order, no early termination: every
// covering Gaussian contributes.  Terms are summed in ascending gid (the key
// order within a tile), so the image is deterministic run-to-run.
// FP32 + MUFU bound; see raster_common.cuh for the CTA layout.
#include "raster_common.cuh"

namespace gi {
namespace {

__global__ void __launch_bounds__(256) render_kernel(const Proj* __restrict__ proj,
                                                     const uint32_t* __restrict__ key_gid,
                                                     const uint32_t* __restrict__ tile_range,
                                                     int W, int H, int T, int TX,
                                                     float* __restrict__ image) {
    __shared__ StagedRecords sr;
    const TileCtx t = make_tile_ctx(W, H, TX);
    const uint32_t s = tile_range[t.img * T + t.tile];
    const uint32_t e = tile_range[t.img * T + t.tile + 1];
    float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f;
    for (uint32_t base = s; base < e; base += 256) {
        const int cnt = (int)min(256u, e - base);
        __syncthreads();
        stage_record(sr, proj, key_gid, base, cnt, t, nullptr);
        __syncthreads();
#pragma unroll 1
        for (int q = 0; q < cnt; q += 32) {
            const int jl = q + t.lane;
            const bool ov = jl < cnt && warp_overlaps(sr.c[jl], t);
            unsigned m = __ballot_sync(kFull, ov);
            while (m) {
                const int j = q + __ffs(m) - 1;
                m &= m - 1;
                const float4 A = sr.a[j];
                const float4 B = sr.b[j];
                const int4 Cb = sr.c[j];
                const PairEval pe = eval_pair(A, B, t);
                const float w = pixel_in_box(Cb, t) ? pe.w : 0.f;
                acc0 = fmaf(B.y, w, acc0);
                acc1 = fmaf(B.z, w, acc1);
                acc2 = fmaf(B.w, w, acc2);
            }
        }
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

cudaError_t launch_render(const Proj* proj, const uint32_t* key_gid, const uint32_t* tile_range,
                          int n, const gi_frame& f, float* image, cudaStream_t s) {
    (void)n;
    const int TX = tiles_x(f.width), T = TX * tiles_y(f.height);
    dim3 grid(T, f.batch);
    render_kernel<<<grid, 256, 0, s>>>(proj, key_gid, tile_range, f.width, f.height, T, TX, image);
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace gi
