// NEXT-2 attribute quantisation of one Gaussian (the encoder of gi.h), shared
// by gi_vq_encode and the QAT step.  Every arithmetic step that decides a code
// is an explicitly rounded fp32 intrinsic (no FMA contraction), so the codes
// are the same function of the inputs as the oracle's.
#pragma once
#include <cuda_fp16.h>

#include "gi_internal.cuh"

namespace gi {

constexpr int kMaxBook = 8 * 256 * 3;   // stages <= 8, codebook <= 256

struct QuantParams {
    int bits, stages, codebook, ib;
    float gamma[3], beta[3];
};

// a6. Decode record r of the payload (record layout
// SPEC.md:404, reading R21) into the parameter records p0 = {u_x, u_y, l1, l2},
// p1 = {l3, c'}: binary16 positions (exact in fp32), l_i = code_i gamma_i +
// beta_i (Eq. 8, one fp32 rounding), c' = C^1[i^1] + ... (Eq. 9, fp32, stage
// order).  R <= 64-bit records are read through a 72-bit big-endian window;
// sb = the codebooks (stages x codebook x 3 floats), staged in shared memory.
__device__ __forceinline__ void decode_one(const uint8_t* __restrict__ payload, int r, int rec_bits,
                                           const QuantParams& qp, const float* sb, float4& p0,
                                           float4& p1) {
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
    const float l1 = __fmaf_rn((float)take(qp.bits), qp.gamma[0], qp.beta[0]);
    const float l2 = __fmaf_rn((float)take(qp.bits), qp.gamma[1], qp.beta[1]);
    const float l3 = __fmaf_rn((float)take(qp.bits), qp.gamma[2], qp.beta[2]);
    float c0 = 0.f, c1 = 0.f, c2 = 0.f;
    for (int m = 0; m < qp.stages; ++m) {
        // an ib-bit field can exceed B - 1 when B is not a power of two (a
        // corrupt payload): clamp, so no read leaves the staged codebooks
        const uint32_t idx = min(take(qp.ib), (uint32_t)(qp.codebook - 1));
        const float* cw = sb + (m * qp.codebook + (int)idx) * 3;
        if (m == 0) {
            c0 = cw[0]; c1 = cw[1]; c2 = cw[2];
        } else {
            c0 = __fadd_rn(c0, cw[0]); c1 = __fadd_rn(c1, cw[1]); c2 = __fadd_rn(c2, cw[2]);
        }
    }
    p0 = make_float4(ux, uy, l1, l2);
    p1 = make_float4(l3, c0, c1, c2);
}

// Codec source of the fused decode + projection (gi_decode_render_frame).
struct DecodeSrc {
    const uint8_t* payload;
    const float* books;       // device [stages][codebook][3]
    int rec_bits;
    QuantParams qp;
    float4* params_out;       // decoded records [n][8], or null
};

// Returns the record (MSB-first, 32 + 3 bits + stages ib bits) and the
// dequantised parameters e0, e1 (= what vq_decode returns); on_stage(m, i^m,
// residual r = c' - c^^{m-1}, C^m[i^m]) is called per RVQ stage.
template <class OnStage>
__device__ __forceinline__ uint64_t encode_one(const float4 p0, const float4 p1, bool logit,
                                               const QuantParams& qp, const float* sb, float4& e0,
                                               float4& e1, OnStage on_stage) {
    const double ux = logit ? tanh((double)p0.x) : (double)p0.x;
    const double uy = logit ? tanh((double)p0.y) : (double)p0.y;
    const __half hx = __float2half_rn(__double2float_rn(ux));
    const __half hy = __float2half_rn(__double2float_rn(uy));
    const float qmax = (float)((1u << qp.bits) - 1u);
    const float l[3] = {p0.z, p0.w, p1.x};
    uint32_t code[3];
    float lq[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        float x = __fdiv_rn(__fsub_rn(l[j], qp.beta[j]), qp.gamma[j]);
        x = fminf(fmaxf(x, 0.0f), qmax);
        code[j] = __float2uint_rn(x);
        lq[j] = __fmaf_rn((float)code[j], qp.gamma[j], qp.beta[j]);
    }
    uint64_t v = ((uint64_t)__half_as_ushort(hx) << 16) | (uint64_t)__half_as_ushort(hy);
#pragma unroll
    for (int j = 0; j < 3; ++j) v = (v << qp.bits) | code[j];
    const float c[3] = {p1.y, p1.z, p1.w};
    float ch0 = 0.f, ch1 = 0.f, ch2 = 0.f;
    for (int m = 0; m < qp.stages; ++m) {
        const float r0 = __fsub_rn(c[0], ch0), r1 = __fsub_rn(c[1], ch1), r2 = __fsub_rn(c[2], ch2);
        int best = 0;
        float bestd = __int_as_float(0x7f800000);
        for (int k = 0; k < qp.codebook; ++k) {
            const float* cw = sb + (m * qp.codebook + k) * 3;
            const float d0 = __fsub_rn(cw[0], r0), d1 = __fsub_rn(cw[1], r1), d2 = __fsub_rn(cw[2], r2);
            float dd = __fmul_rn(d0, d0);
            dd = __fadd_rn(dd, __fmul_rn(d1, d1));
            dd = __fadd_rn(dd, __fmul_rn(d2, d2));
            if (dd < bestd) {
                bestd = dd;
                best = k;
            }
        }
        const float* cw = sb + (m * qp.codebook + best) * 3;
        on_stage(m, best, r0, r1, r2, cw);
        if (m == 0) {
            ch0 = cw[0]; ch1 = cw[1]; ch2 = cw[2];
        } else {
            ch0 = __fadd_rn(ch0, cw[0]); ch1 = __fadd_rn(ch1, cw[1]); ch2 = __fadd_rn(ch2, cw[2]);
        }
        v = (v << qp.ib) | (uint64_t)best;
    }
    e0 = make_float4(__half2float(hx), __half2float(hy), lq[0], lq[1]);
    e1 = make_float4(lq[2], ch0, ch1, ch2);
    return v;
}

}  // namespace gi
