// NEXT-2: attribute quantisation-aware fine-tuning step (
// SPEC quant module; readings R30-R33 in DESIGN.md).  Around the fused
// fit core (project + direct binning -> tile kernel -> finalize, on the
// QUANTISED cloud, positions normalised):
//   qat_quantize_kernel  p -> p^ = Q(p) (codec_core.cuh), per-codeword RVQ
//                        statistics of the residuals and the Eq. 10
//                        commitment sum; CTA 0 advances the step counter and
//                        writes the Adam constants
//   qat_update_kernel    straight-through gradients d/draw from d/dp^ (R32),
//                        Adam on the raw parameters, gamma / beta gradient sums
//   qat_finish_kernel    Adam on gamma / beta, EMA codebooks (R33), losses
// Every cross-Gaussian sum is an integer (fixed-point) atomic sum, so the
// step is deterministic.
#include "codec_core.cuh"

namespace gi {
namespace {

constexpr double kFixR = 1099511627776.0;   // 2^40: residual sums, gamma/beta gradients
constexpr double kFixC = 4294967296.0;      // 2^32: commitment (squared distances)

// Accumulator layout (unsigned long long): [stage][codeword][5] = sum r (3),
// count, sum ||r - C||^2 ; then 6 gradient sums (gamma 0-2, beta 0-2).
__device__ __forceinline__ unsigned long long fix(double x, double scale) {
    return (unsigned long long)__double2ll_rn(x * scale);
}

__global__ void __launch_bounds__(256) qat_quantize_kernel(
    const float4* __restrict__ params, int n, QuantParams qp, const float* __restrict__ qparams,
    const float* __restrict__ books,
    float4* __restrict__ eff, unsigned long long* __restrict__ acc, uint32_t* __restrict__ step,
    float* __restrict__ consts, float lr, float b1, float b2) {
    extern __shared__ unsigned long long dyn[];     // [nb][5] accumulators, then [nb][3] books
    const int nb = qp.stages * qp.codebook;
    uint32_t* sa = reinterpret_cast<uint32_t*>(dyn);   // (lo, hi) pairs
    float* sb = reinterpret_cast<float*>(dyn + (size_t)nb * 5);
#pragma unroll
    for (int j = 0; j < 3; ++j) {          // gamma / beta live on the device (updated each step)
        qp.gamma[j] = qparams[j];
        qp.beta[j] = qparams[3 + j];
    }
    for (int i = threadIdx.x; i < nb * 3; i += blockDim.x) sb[i] = books[i];
    for (int i = threadIdx.x; i < nb * 5 * 2; i += blockDim.x) sa[i] = 0u;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const uint32_t t = *step + 1u;
        *step = t;
        consts[0] = lr;
        consts[1] = (float)(1.0 / (1.0 - pow((double)b1, (double)t)));
        consts[2] = (float)(1.0 / (1.0 - pow((double)b2, (double)t)));
    }
    __syncthreads();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        float4 e0, e1;
        encode_one(params[2 * (size_t)i], params[2 * (size_t)i + 1], true, qp, sb, e0, e1,
                   [&](int m, int k, float r0, float r1, float r2, const float* cw) {
                       uint32_t* a = sa + (m * qp.codebook + k) * 10;
                       shared_add_u64(a + 0, fix(r0, kFixR));
                       shared_add_u64(a + 2, fix(r1, kFixR));
                       shared_add_u64(a + 4, fix(r2, kFixR));
                       atomicAdd(a + 6, 1u);      // counts stay far below 2^32
                       const double d0 = (double)r0 - cw[0], d1 = (double)r1 - cw[1],
                                    d2 = (double)r2 - cw[2];
                       shared_add_u64(a + 8, fix(d0 * d0 + d1 * d1 + d2 * d2, kFixC));
                   });
        eff[2 * (size_t)i] = e0;
        eff[2 * (size_t)i + 1] = e1;
    }
    __syncthreads();
    for (int k = threadIdx.x; k < nb; k += blockDim.x)
        if (shared_read_u64(sa + 10 * k + 6) != 0ull)
            for (int j = 0; j < 5; ++j) atomicAdd(&acc[5 * k + j], shared_read_u64(sa + 10 * k + 2 * j));
}

// gi_adam_step's arithmetic (one definition: adam_update)
__device__ __forceinline__ float adam_step(float p, float g, float& m, float& v, float b1, float b2,
                                           float lr, float ibc1, float ibc2, float eps) {
    return adam_update(p, g, m, v, b1, b2, 1.0f - b1, 1.0f - b2, lr, ibc1, ibc2, eps);
}

// grads holds d/dp^ on entry and d/draw on exit.
__global__ void __launch_bounds__(256) qat_update_kernel(
    float4* __restrict__ params, float4* __restrict__ m, float4* __restrict__ v,
    float4* __restrict__ grads, int n, int bits, const float* __restrict__ qparams,
    const float* __restrict__ consts, float b1, float b2, float eps,
    unsigned long long* __restrict__ gacc, uint32_t* __restrict__ flag) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    double dq[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    if (i < n) {
        float4 p0 = params[2 * (size_t)i], p1 = params[2 * (size_t)i + 1];
        float4 g0 = grads[2 * (size_t)i], g1 = grads[2 * (size_t)i + 1];
        const float qmax = (float)((1u << bits) - 1u);
        const float l[3] = {p0.z, p0.w, p1.x};
        const float ge[3] = {g0.z, g0.w, g1.x};
        float gl[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const float x = __fdiv_rn(__fsub_rn(l[j], qparams[3 + j]), qparams[j]);
            const bool inside = x >= 0.0f && x <= qmax;
            const float code = (float)__float2uint_rn(fminf(fmaxf(x, 0.0f), qmax));
            gl[j] = inside ? ge[j] : 0.0f;
            dq[j] = (double)ge[j] * (inside ? (double)code - (double)x : (double)code);
            dq[3 + j] = inside ? 0.0 : (double)ge[j];
        }
        // positions: u = tanh(raw), d/draw = d/du / cosh^2(raw)
        const float chx = coshf(p0.x), chy = coshf(p0.y);
        g0.x = g0.x / (chx * chx);
        g0.y = g0.y / (chy * chy);
        g0.z = gl[0];
        g0.w = gl[1];
        g1.x = gl[2];
        grads[2 * (size_t)i] = g0;
        grads[2 * (size_t)i + 1] = g1;
        const float lr = consts[0], ibc1 = consts[1], ibc2 = consts[2];
        float4 m0 = m[2 * (size_t)i], m1 = m[2 * (size_t)i + 1];
        float4 v0 = v[2 * (size_t)i], v1 = v[2 * (size_t)i + 1];
        p0.x = adam_step(p0.x, g0.x, m0.x, v0.x, b1, b2, lr, ibc1, ibc2, eps);
        p0.y = adam_step(p0.y, g0.y, m0.y, v0.y, b1, b2, lr, ibc1, ibc2, eps);
        p0.z = adam_step(p0.z, g0.z, m0.z, v0.z, b1, b2, lr, ibc1, ibc2, eps);
        p0.w = adam_step(p0.w, g0.w, m0.w, v0.w, b1, b2, lr, ibc1, ibc2, eps);
        p1.x = adam_step(p1.x, g1.x, m1.x, v1.x, b1, b2, lr, ibc1, ibc2, eps);
        p1.y = adam_step(p1.y, g1.y, m1.y, v1.y, b1, b2, lr, ibc1, ibc2, eps);
        p1.z = adam_step(p1.z, g1.z, m1.z, v1.z, b1, b2, lr, ibc1, ibc2, eps);
        p1.w = adam_step(p1.w, g1.w, m1.w, v1.w, b1, b2, lr, ibc1, ibc2, eps);
        params[2 * (size_t)i] = p0;
        params[2 * (size_t)i + 1] = p1;
        m[2 * (size_t)i] = m0;
        m[2 * (size_t)i + 1] = m1;
        v[2 * (size_t)i] = v0;
        v[2 * (size_t)i + 1] = v1;
        const bool bad = !(isfinite(p0.x) && isfinite(p0.y) && isfinite(p0.z) && isfinite(p0.w) &&
                           isfinite(p1.x) && isfinite(p1.y) && isfinite(p1.z) && isfinite(p1.w));
        if (bad && flag != nullptr) atomicOr(flag, 1u);
    }
    // gamma / beta gradient sums: per-thread contributions to fixed point
    // first (so the total is an integer sum, order-independent), warp sums,
    // one atomic per warp
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < 6; ++j) {
        long long q = __double2ll_rn(dq[j] * kFixR);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(kFull, q, o);
        if (lane == 0 && q != 0) atomicAdd(&gacc[j], (unsigned long long)q);
    }
}

__global__ void qat_finish_kernel(float* __restrict__ qparams, float* __restrict__ qm,
                                  float* __restrict__ qv, float* __restrict__ books,
                                  float* __restrict__ ema_n, float* __restrict__ ema_s,
                                  unsigned long long* __restrict__ acc, int nb, int n, int codebook,
                                  const float* __restrict__ consts, float b1, float b2, float eps,
                                  float decay, float lambda, float* __restrict__ losses) {
    unsigned long long* gacc = acc + 5 * nb;
    if (threadIdx.x < 6) {
        const int j = threadIdx.x;
        const float g = (float)((double)(long long)gacc[j] * (1.0 / kFixR));
        losses[3 + j] = g;                  // d/dgamma_0..2, d/dbeta_0..2 (diagnostic)
        float mm = qm[j], vv = qv[j];
        qparams[j] = adam_step(qparams[j], g, mm, vv, b1, b2, consts[0], consts[1], consts[2], eps);
        qm[j] = mm;
        qv[j] = vv;
        gacc[j] = 0ull;
    }
    __shared__ double commit[256];
    double cs = 0.0;
    for (int k = threadIdx.x; k < nb; k += blockDim.x) {
        unsigned long long* a = acc + 5 * k;
        const double cnt = (double)(long long)a[3];
        cs += (double)(long long)a[4] * (1.0 / kFixC);
        const double en = (double)decay * ema_n[k] + (1.0 - (double)decay) * cnt;
        ema_n[k] = (float)en;
        double es[3];
        for (int j = 0; j < 3; ++j) {
            es[j] = (double)decay * ema_s[3 * k + j] +
                    (1.0 - (double)decay) * ((double)(long long)a[j] * (1.0 / kFixR));
            ema_s[3 * k + j] = (float)es[j];
        }
        if (cnt > 0.0)
            for (int j = 0; j < 3; ++j) books[3 * k + j] = (float)(es[j] / en);
        for (int j = 0; j < 5; ++j) a[j] = 0ull;
    }
    commit[threadIdx.x] = cs;
    __syncthreads();
    if (threadIdx.x == 0) {
        double c = 0.0;
        for (int t = 0; t < (int)blockDim.x; ++t) c += commit[t];
        const double lc = c / ((double)n * (double)codebook);
        losses[2] = (float)lc;
        losses[0] = (float)((double)losses[1] + (double)lambda * lc);
    }
}

}  // namespace

size_t qat_acc_words(int stages, int codebook) { return (size_t)stages * codebook * 5 + 6; }

cudaError_t launch_qat_quantize(const float* params, int n, const QuantParams& qp,
                                const float* qparams, const float* books, float* eff, void* acc,
                                uint32_t* step,
                                float* consts, float lr, float b1, float b2, cudaStream_t s) {
    const size_t nb = (size_t)qp.stages * qp.codebook;
    const size_t smem = nb * 5 * sizeof(unsigned long long) + nb * 3 * sizeof(float);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(qat_quantize_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    qat_quantize_kernel<<<(n + 255) / 256 > 0 ? (n + 255) / 256 : 1, 256, smem, s>>>(
        reinterpret_cast<const float4*>(params), n, qp, qparams, books, reinterpret_cast<float4*>(eff),
        static_cast<unsigned long long*>(acc), step, consts, lr, b1, b2);
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_qat_update(float* params, float* m, float* v, float* grads, int n, int bits,
                              const float* qparams, const float* consts, float b1, float b2,
                              float eps, void* acc, int stages, int codebook, uint32_t* flag,
                              cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    qat_update_kernel<<<(n + 255) / 256, 256, 0, s>>>(
        reinterpret_cast<float4*>(params), reinterpret_cast<float4*>(m),
        reinterpret_cast<float4*>(v), reinterpret_cast<float4*>(grads), n, bits, qparams, consts, b1,
        b2, eps, static_cast<unsigned long long*>(acc) + (size_t)stages * codebook * 5, flag);
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_qat_finish(float* qparams, float* qm, float* qv, float* books, float* ema_n,
                              float* ema_s, void* acc, int stages, int codebook, int n,
                              const float* consts, float b1, float b2, float eps, float decay,
                              float lambda, float* losses, cudaStream_t s) {
    qat_finish_kernel<<<1, 256, 0, s>>>(qparams, qm, qv, books, ema_n, ema_s,
                                        static_cast<unsigned long long*>(acc), stages * codebook, n,
                                        codebook, consts, b1, b2, eps, decay, lambda, losses);
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace gi
