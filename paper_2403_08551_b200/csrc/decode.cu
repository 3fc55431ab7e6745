// a6. Attribute decode of the codec path (Table 2 decode
// FPS P:426; record layout SPEC.md:404, reading R21):
//   u = binary16 position (R19)          -> exact fp32
//   l_i = code_i * gamma_i + beta_i  (Eq. 8)    -> one fp32 rounding (fmaf)
//   c' = C^1[i^1] + ... + C^M[i^M]  (Eq. 9)     -> fp32, stage order
// One thread per record; R <= 64-bit records are read through a 72-bit
// big-endian window; codebooks (M*B*3 floats) are staged in shared memory.
// Output feeds gi_project(GI_POS_NORMALIZED).
#include <cuda_fp16.h>

#include "gi_internal.cuh"

namespace gi {
namespace {

constexpr int kMaxBook = 8 * 256 * 3;   // stages <= 8, codebook <= 256

__global__ void __launch_bounds__(256) vq_decode_kernel(const uint8_t* __restrict__ payload,
                                                        int n, int bits, int stages, int codebook,
                                                        int ib, int rec_bits, float g0, float g1,
                                                        float g2, float b0, float b1, float b2,
                                                        const float* __restrict__ books,
                                                        float4* __restrict__ params) {
    __shared__ float sb[kMaxBook];
    const int nb = stages * codebook * 3;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) sb[i] = books[i];
    __syncthreads();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int64_t bit0 = (int64_t)r * rec_bits;
    const int64_t byte0 = bit0 >> 3;
    const int sh = (int)(bit0 & 7);
    const int nbytes = (sh + rec_bits + 7) >> 3;      // bytes the record touches (<= 9)
    uint64_t hi = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) hi = (hi << 8) | (i < nbytes ? (uint64_t)payload[byte0 + i] : 0ull);
    const uint64_t extra = nbytes > 8 ? (uint64_t)payload[byte0 + 8] : 0ull;
    // window: the record's bits start at the MSB
    const uint64_t win = sh ? ((hi << sh) | (extra >> (8 - sh))) : hi;
    int pos = 0;
    auto take = [&](int width) -> uint32_t {
        const uint32_t v = (uint32_t)((win << pos) >> (64 - width));
        pos += width;
        return v;
    };
    const uint32_t hx = take(16), hy = take(16);
    const float ux = __half2float(__ushort_as_half((unsigned short)hx));
    const float uy = __half2float(__ushort_as_half((unsigned short)hy));
    const float l1 = __fmaf_rn((float)take(bits), g0, b0);
    const float l2 = __fmaf_rn((float)take(bits), g1, b1);
    const float l3 = __fmaf_rn((float)take(bits), g2, b2);
    float c0 = 0.f, c1 = 0.f, c2 = 0.f;
    for (int m = 0; m < stages; ++m) {
        const uint32_t idx = take(ib);
        const float* cw = sb + (m * codebook + (int)idx) * 3;
        if (m == 0) {
            c0 = cw[0]; c1 = cw[1]; c2 = cw[2];
        } else {
            c0 = __fadd_rn(c0, cw[0]); c1 = __fadd_rn(c1, cw[1]); c2 = __fadd_rn(c2, cw[2]);
        }
    }
    params[2 * (size_t)r] = make_float4(ux, uy, l1, l2);
    params[2 * (size_t)r + 1] = make_float4(l3, c0, c1, c2);
}

}  // namespace

cudaError_t launch_vq_decode(const uint8_t* payload, const gi_codec_meta& meta, float* params,
                             cudaStream_t s) {
    if (meta.n == 0) return cudaSuccess;
    int ib = 1;
    while ((1 << ib) < meta.codebook) ++ib;
    const int rec = 32 + 3 * meta.bits + meta.stages * ib;
    vq_decode_kernel<<<(meta.n + 255) / 256, 256, 0, s>>>(
        payload, meta.n, meta.bits, meta.stages, meta.codebook, ib, rec, meta.gamma[0],
        meta.gamma[1], meta.gamma[2], meta.beta[0], meta.beta[1], meta.beta[2], meta.codebooks,
        reinterpret_cast<float4*>(params));
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace gi
