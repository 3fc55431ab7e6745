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
