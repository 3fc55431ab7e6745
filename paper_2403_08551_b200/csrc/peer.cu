// NEXT-4: the gradient exchange of single-image spatial
// sharding fused with the optimiser.  Every rank renders and back-propagates
// its own tile rows (gi_fit_grads) into an exchange buffer that the other
// ranks of the node have mapped (CUDA IPC, NVLink peer access); one kernel on
// each rank then reads all G buffers, sums them in rank order -- the same
// order on every rank, so the replicas stay bit-identical -- and applies
// Adam (the arithmetic of gi_adam_step: adam_update).  This replaces the
// all-reduce + optimiser pair: the gradient bytes cross NVLink once, inside
// the kernel that consumes them.  Element-wise, float4 vectorised: G loads of
// 16 B per 4 scalars + the Adam traffic (28 B per scalar).
#include "gi_internal.cuh"

namespace gi {
namespace {

struct PeerPtrs {
    const float* g[kMaxPeers];
    int G;
};

__device__ __forceinline__ float4 peer_sum4(const PeerPtrs& pp, int64_t i) {
    float4 s = reinterpret_cast<const float4*>(pp.g[0])[i];
    for (int r = 1; r < pp.G; ++r) {
        const float4 x = reinterpret_cast<const float4*>(pp.g[r])[i];
        s.x += x.x; s.y += x.y; s.z += x.z; s.w += x.w;
    }
    return s;
}

// the bias corrections exactly as adam_kernel forms them (fp64 pow on the
// device, rounded once)
__device__ __forceinline__ void bias_corrections(int t, float b1, float b2, float& ibc1, float& ibc2) {
    ibc1 = (float)(1.0 / (1.0 - pow((double)b1, (double)t)));
    ibc2 = (float)(1.0 / (1.0 - pow((double)b2, (double)t)));
}

__global__ void __launch_bounds__(256) peer_adam_kernel(float4* __restrict__ p, float4* __restrict__ m,
                                                        float4* __restrict__ v, PeerPtrs pp,
                                                        int64_t count4, int step, float lr, float b1,
                                                        float b2, float eps, uint32_t* flag) {
    __shared__ float sconst[2];
    if (threadIdx.x == 0) bias_corrections(step, b1, b2, sconst[0], sconst[1]);
    __syncthreads();
    const float ibc1 = sconst[0], ibc2 = sconst[1];
    const float omb1 = 1.0f - b1, omb2 = 1.0f - b2;
    bool bad = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count4;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float4 gg = peer_sum4(pp, i);
        float4 q = p[i], mm = m[i], vv = v[i];
        bad |= !isfinite(adam_update(q.x, gg.x, mm.x, vv.x, b1, b2, omb1, omb2, lr, ibc1, ibc2, eps));
        bad |= !isfinite(adam_update(q.y, gg.y, mm.y, vv.y, b1, b2, omb1, omb2, lr, ibc1, ibc2, eps));
        bad |= !isfinite(adam_update(q.z, gg.z, mm.z, vv.z, b1, b2, omb1, omb2, lr, ibc1, ibc2, eps));
        bad |= !isfinite(adam_update(q.w, gg.w, mm.w, vv.w, b1, b2, omb1, omb2, lr, ibc1, ibc2, eps));
        p[i] = q;
        m[i] = mm;
        v[i] = vv;
    }
    if (flag != nullptr && __any_sync(kFull, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

// scalar tail of the parameters (count % 4) and the loss floats
__global__ void peer_tail_kernel(float* p, float* m, float* v, PeerPtrs pp, int64_t start,
                                 int64_t count, int step, float lr, float b1, float b2, float eps,
                                 int n_loss, float* loss_out, uint32_t* flag) {
    const int64_t i = start + threadIdx.x;
    if (i < count) {
        float ibc1, ibc2;
        bias_corrections(step, b1, b2, ibc1, ibc2);
        float g = pp.g[0][i];
        for (int r = 1; r < pp.G; ++r) g += pp.g[r][i];
        float q = p[i], mm = m[i], vv = v[i];
        if (!isfinite(adam_update(q, g, mm, vv, b1, b2, 1.0f - b1, 1.0f - b2, lr, ibc1, ibc2, eps)) &&
            flag)
            atomicOr(flag, 1u);
        p[i] = q;
        m[i] = mm;
        v[i] = vv;
    }
    if ((int)threadIdx.x < n_loss && loss_out != nullptr) {
        float l = pp.g[0][count + threadIdx.x];
        for (int r = 1; r < pp.G; ++r) l += pp.g[r][count + threadIdx.x];
        loss_out[threadIdx.x] = l;
    }
}

}  // namespace

cudaError_t launch_peer_adam(float* params, float* m, float* v, const float* const* grads, int G,
                             int64_t count, int step, float lr, float b1, float b2, float eps,
                             int n_loss, float* loss_out, uint32_t* flag, cudaStream_t s) {
    PeerPtrs pp{};
    pp.G = G;
    for (int r = 0; r < G; ++r) pp.g[r] = grads[r];
    const int64_t c4 = count / 4;
    if (c4 > 0) {
        int64_t blocks = (c4 + 255) / 256;
        if (blocks > 148 * 16) blocks = 148 * 16;
        peer_adam_kernel<<<(unsigned)blocks, 256, 0, s>>>(
            reinterpret_cast<float4*>(params), reinterpret_cast<float4*>(m),
            reinterpret_cast<float4*>(v), pp, c4, step, lr, b1, b2, eps, flag);
        note_launches(1);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    if (count % 4 != 0 || n_loss > 0) {
        peer_tail_kernel<<<1, 32, 0, s>>>(params, m, v, pp, c4 * 4, count, step, lr, b1, b2, eps,
                                          n_loss, loss_out, flag);
        note_launches(1);
    }
    return cudaGetLastError();
}

}  // namespace gi
