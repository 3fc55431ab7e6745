// a5. Adam (north_star "feeding an Adam fitting loop"; reading R16) with the
// paper's schedule lr_t = lr0 * 0.5^floor((t-1)/20000) (R17).
// Elementwise over the AoS parameter array, float4 vectorised: 28 B of HBM/L2
// traffic per scalar (read p, g, m, v; write p, m, v).  The bias corrections
// 1 - beta^t are formed once per CTA in fp64.
#include "gi_internal.cuh"

namespace gi {
namespace {

__device__ __forceinline__ float adam1(float& p, float g, float& m, float& v, float b1, float b2,
                                       float omb1, float omb2, float lr, float ibc1, float ibc2,
                                       float eps) {
    return adam_update(p, g, m, v, b1, b2, omb1, omb2, lr, ibc1, ibc2, eps);
}

__global__ void __launch_bounds__(256) adam_kernel(float4* __restrict__ p, const float4* __restrict__ g,
                                                   float4* __restrict__ m, float4* __restrict__ v,
                                                   int64_t count4, int step, const uint32_t* step_dev,
                                                   float lr, int half_every, float b1, float b2,
                                                   float eps, uint32_t* flag) {
    __shared__ float sconst[3];
    if (threadIdx.x == 0) {
        const int t = step_dev ? (int)*step_dev : step;
        float lr_t = lr;
        if (step_dev) lr_t = ldexpf(lr, -((t - 1) / half_every));   // exact power-of-2 halving
        sconst[0] = lr_t;
        sconst[1] = (float)(1.0 / (1.0 - pow((double)b1, (double)t)));
        sconst[2] = (float)(1.0 / (1.0 - pow((double)b2, (double)t)));
    }
    __syncthreads();
    const float lr_t = sconst[0], ibc1 = sconst[1], ibc2 = sconst[2];
    const float omb1 = 1.0f - b1, omb2 = 1.0f - b2;
    bool bad = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count4;
         i += (int64_t)gridDim.x * blockDim.x) {
        float4 pp = p[i], mm = m[i], vv = v[i];
        const float4 gg = g[i];
        bad |= !isfinite(adam1(pp.x, gg.x, mm.x, vv.x, b1, b2, omb1, omb2, lr_t, ibc1, ibc2, eps));
        bad |= !isfinite(adam1(pp.y, gg.y, mm.y, vv.y, b1, b2, omb1, omb2, lr_t, ibc1, ibc2, eps));
        bad |= !isfinite(adam1(pp.z, gg.z, mm.z, vv.z, b1, b2, omb1, omb2, lr_t, ibc1, ibc2, eps));
        bad |= !isfinite(adam1(pp.w, gg.w, mm.w, vv.w, b1, b2, omb1, omb2, lr_t, ibc1, ibc2, eps));
        p[i] = pp;
        m[i] = mm;
        v[i] = vv;
    }
    if (flag != nullptr && __any_sync(kFull, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

// scalar tail (count not a multiple of 4)
__global__ void adam_tail_kernel(float* p, const float* g, float* m, float* v, int64_t start,
                                 int64_t count, int step, const uint32_t* step_dev, float lr,
                                 int half_every, float b1, float b2, float eps, uint32_t* flag) {
    const int64_t i = start + threadIdx.x;
    if (i >= count) return;
    const int t = step_dev ? (int)*step_dev : step;
    const float lr_t = step_dev ? ldexpf(lr, -((t - 1) / half_every)) : lr;
    const float ibc1 = (float)(1.0 / (1.0 - pow((double)b1, (double)t)));
    const float ibc2 = (float)(1.0 / (1.0 - pow((double)b2, (double)t)));
    float pp = p[i], mm = m[i], vv = v[i];
    if (!isfinite(adam1(pp, g[i], mm, vv, b1, b2, 1.0f - b1, 1.0f - b2, lr_t, ibc1, ibc2, eps)) && flag)
        atomicOr(flag, 1u);
    p[i] = pp;
    m[i] = mm;
    v[i] = vv;
}

}  // namespace

cudaError_t launch_adam(float* params, const float* grads, float* m, float* v, int64_t count,
                        int step, const uint32_t* step_dev, float lr, int half_every, float b1,
                        float b2, float eps, uint32_t* flag, cudaStream_t s) {
    const int64_t c4 = count / 4;
    if (c4 > 0) {
        int64_t blocks = (c4 + 255) / 256;
        if (blocks > 148 * 16) blocks = 148 * 16;
        adam_kernel<<<(unsigned)blocks, 256, 0, s>>>(
            reinterpret_cast<float4*>(params), reinterpret_cast<const float4*>(grads),
            reinterpret_cast<float4*>(m), reinterpret_cast<float4*>(v), c4, step, step_dev, lr,
            half_every, b1, b2, eps, flag);
        note_launches(1);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    if (count % 4) {
        adam_tail_kernel<<<1, 32, 0, s>>>(params, grads, m, v, c4 * 4, count, step, step_dev, lr,
                                          half_every, b1, b2, eps, flag);
        note_launches(1);
    }
    return cudaGetLastError();
}

}  // namespace gi
