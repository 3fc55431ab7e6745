// NEXT-1: the paper's optimiser, Adan ("optimized over 50000
// steps using the Adan optimizer"; the update rule is the cited Adan
// reference's, hyper-parameters per SPEC.md:231 -- reading R28):
//   d = g - g_prev            (0 at step 1)
//   m = b1 m + (1-b1) g;  v = b2 v + (1-b2) d;  n = b3 n + (1-b3) (g + b2 d)^2
//   p = p (1 - lr wd) - lr (m/(1-b1^t) + b2 v/(1-b2^t)) / (sqrt(n/(1-b3^t)) + eps)
//   g_prev = g
// Elementwise over the AoS parameters, float4 vectorised (44 B of traffic per
// scalar); the step t and lr_t = lr0 * 0.5^floor((t-1)/half_every) come from
// the host or from the device step counter (graph capture).
#include "gi_internal.cuh"

namespace gi {
namespace {

__global__ void __launch_bounds__(256) adan_kernel(float4* __restrict__ p, const float4* __restrict__ g,
                                                   float4* __restrict__ m, float4* __restrict__ v,
                                                   float4* __restrict__ n, float4* __restrict__ gp,
                                                   int64_t count4, int step, const uint32_t* step_dev,
                                                   float lr, int half_every, float b1, float b2,
                                                   float b3, float eps, float wd, uint32_t* flag) {
    __shared__ AdanConsts sc;
    griddep_wait();
    griddep_trigger();
    if (threadIdx.x == 0) {
        const int t = step_dev ? (int)*step_dev : step;
        const float lr_t = step_dev ? ldexpf(lr, -((t - 1) / half_every)) : lr;
        sc.lr = lr_t;
        sc.ibc1 = (float)(1.0 / (1.0 - pow((double)b1, (double)t)));
        sc.ibc2 = (float)(1.0 / (1.0 - pow((double)b2, (double)t)));
        sc.isbc3 = (float)(1.0 / sqrt(1.0 - pow((double)b3, (double)t)));
        sc.b1 = b1; sc.b2 = b2; sc.b3 = b3; sc.eps = eps;
        sc.decay = 1.0f - lr_t * wd;
        sc.first = t == 1;
    }
    __syncthreads();
    const AdanConsts c = sc;
    bool bad = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count4;
         i += (int64_t)gridDim.x * blockDim.x) {
        float4 pp = p[i], mm = m[i], vv = v[i], nn = n[i], pg = gp[i];
        const float4 gg = g[i];
        pp.x = adan1(pp.x, gg.x, mm.x, vv.x, nn.x, pg.x, c);
        pp.y = adan1(pp.y, gg.y, mm.y, vv.y, nn.y, pg.y, c);
        pp.z = adan1(pp.z, gg.z, mm.z, vv.z, nn.z, pg.z, c);
        pp.w = adan1(pp.w, gg.w, mm.w, vv.w, nn.w, pg.w, c);
        bad |= !(isfinite(pp.x) && isfinite(pp.y) && isfinite(pp.z) && isfinite(pp.w));
        p[i] = pp; m[i] = mm; v[i] = vv; n[i] = nn; gp[i] = pg;
    }
    if (flag != nullptr && __any_sync(kFull, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

}  // namespace

cudaError_t launch_adan(float* params, const float* grads, float* m, float* v, float* n,
                        float* gprev, int64_t count, int step, const uint32_t* step_dev, float lr,
                        int half_every, float b1, float b2, float b3, float eps, float wd,
                        uint32_t* flag, cudaStream_t s) {
    const int64_t c4 = count / 4;       // count is a multiple of 8 (AoS [N][8])
    if (c4 == 0) return cudaSuccess;
    int64_t blocks = (c4 + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    cudaError_t e = launch_pdl(adan_kernel, dim3((unsigned)blocks), dim3(256), s,
                               reinterpret_cast<float4*>(params), reinterpret_cast<const float4*>(grads),
                               reinterpret_cast<float4*>(m), reinterpret_cast<float4*>(v),
                               reinterpret_cast<float4*>(n), reinterpret_cast<float4*>(gprev), c4, step,
                               step_dev, lr, half_every, b1, b2, b3, eps, wd, flag);
    note_launches(1);
    return e;
}

}  // namespace gi
