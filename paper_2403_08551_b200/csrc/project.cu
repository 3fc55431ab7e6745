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
// float -> int decisions are reproducible.  The conic is formed in fp64 and
// rounded once.
#include "project_core.cuh"

namespace gi {
namespace {

__global__ void __launch_bounds__(256) project_kernel(const float4* __restrict__ params, int n,
                                                      int total, int W, int H, float k,
                                                      uint32_t flags, Proj* __restrict__ proj,
                                                      uint32_t* __restrict__ tiles_touched,
                                                      ProjectFuse fuse) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g < total) prefetch_l2(params + 2 * (size_t)g);   // 32 B record; safe before the wait
    griddep_wait();
    griddep_trigger();
    if (fuse.step_counter != nullptr && g == 0) *fuse.step_counter += 1u;   // fused fit: t <- t + 1
    uint32_t touched = 0;
    int4 rect = make_int4(0, -1, 0, -1);
    if (g < total) {
        touched = project_one(params[2 * (size_t)g], params[2 * (size_t)g + 1], g, n, W, H, k,
                              flags, proj, fuse.counts, rect);
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
    const int blocks = (total + 255) / 256;
    if (blocks == 0 && fuse.step_counter == nullptr) return cudaSuccess;
    launch_pdl(project_kernel, dim3(blocks > 0 ? blocks : 1), dim3(256), s,
               reinterpret_cast<const float4*>(params), n, total, f.width, f.height, f.k, flags, proj,
               tiles_touched, fuse);
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace gi
