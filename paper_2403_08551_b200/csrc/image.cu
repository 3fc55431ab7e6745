// Fit targets from 8-bit RGB images.  The paper's datasets -- Kodak (24
// images, 768x512) and DIV2K -- are 24-bit RGB images; a caller that
// holds one decoded (interleaved [B][H][W][3] u8) moves it across the host
// link at one byte per channel (1.18 MB for a Kodak image instead of 4.72 MB
// of fp32) and this kernel writes the planar [B][3][H][W] fp32 target the fit
// kernels read, value u / 255 (IEEE division, round to nearest: bit-exact
// with numpy's float32(u) / float32(255)).
#include "gi_internal.cuh"

namespace gi {
namespace {

// one thread per pixel: 3 bytes in (a warp reads 96 contiguous bytes), one
// float per plane out (coalesced per plane)
__global__ void __launch_bounds__(256) rgb8_kernel(const uint8_t* __restrict__ rgb, int64_t P,
                                                   float* __restrict__ target) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    const size_t img = blockIdx.y;
    const uint8_t* s = rgb + img * 3 * (size_t)P + 3 * (size_t)p;
    float* d = target + img * 3 * (size_t)P + (size_t)p;
    const float r = __fdiv_rn((float)s[0], 255.0f);
    const float g = __fdiv_rn((float)s[1], 255.0f);
    const float b = __fdiv_rn((float)s[2], 255.0f);
    d[0] = r;
    d[P] = g;
    d[2 * P] = b;
}

}  // namespace

cudaError_t launch_target_from_rgb8(const uint8_t* rgb, const gi_frame& f, float* target,
                                    cudaStream_t s) {
    const int64_t P = (int64_t)f.width * f.height;
    if (P == 0 || f.batch == 0) return cudaSuccess;
    const dim3 grid((unsigned)((P + 255) / 256), (unsigned)f.batch);
    rgb8_kernel<<<grid, 256, 0, s>>>(rgb, P, target);
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace gi
