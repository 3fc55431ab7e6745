// a1. Projection ("formation"; Eq. 1; App. C).
//
// One thread per Gaussian, two coalesced float4 loads of the AoS parameters,
// three float4 stores of the 48-byte record.  HBM/L2-bound: 32 B in,
// 52 B out per Gaussian.
//
// Precision plan: tanh and the pixel-space centre
// are computed in fp64 and split into an integer pixel plus an fp32 fraction
// (an fp32 centre near x = 768 has an ulp of 6e-5 px, which alone breaks the
// 2e-5 pixel bar).  The box is decided by the fp32 recipe of reading R7 with
// explicitly rounded intrinsics (no FMA contraction), so that its
// float -> int decisions are reproducible.  The Cholesky conic is formed by
// IEEE fp32 divisions (a = kappa / l1e, c = kappa / l3e, b = -(a l2) / l3e:
// < 1e-6 relative on sigma near the box edge); the RS conic from the fp64
// Cholesky factor of Sigma, rounded once.
#include "codec_core.cuh"
#include "project_core.cuh"

namespace gi {
namespace {

// kDecode (gi_decode_render_frame): the parameters come from decoding record
// g of the codec payload (decode_one, codebooks staged in dynamic shared
// memory) instead of a load -- a6 and a1 in one pass, no parameter round trip.
template <bool kDecode>
#ifndef GI_PROJ_THREADS
#define GI_PROJ_THREADS 256
#endif
__global__ void __launch_bounds__(GI_PROJ_THREADS) project_kernel(const float4* __restrict__ params, int n,
                                                      int total, int W, int H, float k,
                                                      uint32_t flags, Proj* __restrict__ proj,
                                                      uint32_t* __restrict__ tiles_touched,
                                                      ProjectFuse fuse, DecodeSrc dec) {
    extern __shared__ float sbook[];
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (!kDecode && g < total) prefetch_l2(params + 2 * (size_t)g);   // 32 B record; safe before the wait
    griddep_wait();
    griddep_trigger();
    if constexpr (kDecode) {
        const int nb = dec.qp.stages * dec.qp.codebook * 3;
        for (int i = threadIdx.x; i < nb; i += blockDim.x) sbook[i] = dec.books[i];
        __syncthreads();
    }
    if (fuse.step_counter != nullptr && g == 0) *fuse.step_counter += 1u;   // fused fit: t <- t + 1
    uint32_t touched = 0;
    int4 rect = make_int4(0, -1, 0, -1);
    if (g < total) {
        float4 p0, p1;
        if constexpr (kDecode) {
            decode_one(dec.payload, g, dec.rec_bits, dec.qp, sbook, p0, p1);
            if (dec.params_out != nullptr) {
                dec.params_out[2 * (size_t)g] = p0;
                dec.params_out[2 * (size_t)g + 1] = p1;
            }
        } else {
            p0 = params[2 * (size_t)g];
            p1 = params[2 * (size_t)g + 1];
        }
        touched = project_one(p0, p1, g, n, W, H, k, flags, proj, fuse.counts, rect);
        tiles_touched[g] = touched;
    }
    if (fuse.counts.tile_count != nullptr) {
        const int TX = (W + kTile - 1) / kTile;
        const int T = TX * (fuse.counts.row1 > 0 ? fuse.counts.row1 - fuse.counts.row0
                                                 : (H + kTile - 1) / kTile);
        post_project_warp(fuse.counts, touched, rect, g, g < total ? (g / n) * T : 0, TX, total);
    }
}

}  // namespace

cudaError_t launch_project(const float* params, int n, const gi_frame& f, uint32_t flags,
                           Proj* proj, uint32_t* tiles_touched, const ProjectFuse& fuse,
                           cudaStream_t s) {
    const int total = n * f.batch;
    const int blocks = (total + GI_PROJ_THREADS - 1) / GI_PROJ_THREADS;
    if (blocks == 0 && fuse.step_counter == nullptr) return cudaSuccess;
    launch_pdl(project_kernel<false>, dim3(blocks > 0 ? blocks : 1), dim3(GI_PROJ_THREADS), s,
               reinterpret_cast<const float4*>(params), n, total, f.width, f.height, f.k, flags, proj,
               tiles_touched, fuse, DecodeSrc{});
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_decode_project(const uint8_t* payload, const gi_codec_meta& meta,
                                  float* params_out, const gi_frame& f, Proj* proj,
                                  uint32_t* tiles_touched, const ProjectFuse& fuse, cudaStream_t s) {
    const int n = meta.n;
    const int blocks = (n + GI_PROJ_THREADS - 1) / GI_PROJ_THREADS;
    if (blocks == 0) return cudaSuccess;
    int ib = 1;
    while ((1 << ib) < meta.codebook) ++ib;
    DecodeSrc dec{payload, meta.codebooks, 32 + 3 * meta.bits + meta.stages * ib,
                  QuantParams{meta.bits, meta.stages, meta.codebook, ib,
                              {meta.gamma[0], meta.gamma[1], meta.gamma[2]},
                              {meta.beta[0], meta.beta[1], meta.beta[2]}},
                  reinterpret_cast<float4*>(params_out)};
    const size_t smem = (size_t)meta.stages * meta.codebook * 3 * sizeof(float);
    launch_pdl_smem(project_kernel<true>, dim3(blocks), dim3(GI_PROJ_THREADS), smem, s,
                    static_cast<const float4*>(nullptr), n, n, f.width, f.height, f.k,
                    (uint32_t)GI_POS_NORMALIZED, proj, tiles_touched, fuse, dec);
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace gi
