// a6. Attribute decode of the codec path (Table 2 decode
// FPS P:426; record layout SPEC.md:404, reading R21): one thread per record
// (codec_core.cuh: decode_one), codebooks (M*B*3 floats) staged in shared
// memory.  Output feeds gi_project(GI_POS_NORMALIZED); gi_decode_render_frame
// fuses the same decode into the projection kernel (project.cu).
#include "codec_core.cuh"

namespace gi {
namespace {

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
    const QuantParams qp{bits, stages, codebook, ib, {g0, g1, g2}, {b0, b1, b2}};
    float4 p0, p1;
    decode_one(payload, r, rec_bits, qp, sb, p0, p1);
    params[2 * (size_t)r] = p0;
    params[2 * (size_t)r + 1] = p1;
}

// NEXT-2 encoder (the inverse of vq_decode_kernel; see gi.h): one thread per
// Gaussian.  Every arithmetic step that decides a code is an explicitly
// rounded fp32 intrinsic (no FMA contraction), so the codes are the same
// function of the inputs as the oracle's.  Records are written MSB-first:
// with whole-byte records (the paper's 56-bit default) by plain byte stores,
// otherwise by atomicOr into the 32-bit words they straddle (the payload is
// zero-filled first; OR is order-independent, so the result is
// deterministic).
__global__ void __launch_bounds__(256) vq_encode_kernel(
    const float4* __restrict__ params, int n, bool logit, int bits, int stages, int codebook, int ib,
    int rec_bits, float g0, float g1, float g2, float b0, float b1, float b2,
    const float* __restrict__ books, uint8_t* __restrict__ payload, float4* __restrict__ eff) {
    __shared__ float sb[kMaxBook];
    const int nb = stages * codebook * 3;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) sb[i] = books[i];
    __syncthreads();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const QuantParams qp{bits, stages, codebook, ib, {g0, g1, g2}, {b0, b1, b2}};
    float4 e0, e1;
    const uint64_t v = encode_one(params[2 * (size_t)r], params[2 * (size_t)r + 1], logit, qp, sb,
                                  e0, e1, [](int, int, float, float, float, const float*) {});
    if (eff != nullptr) {
        eff[2 * (size_t)r] = e0;
        eff[2 * (size_t)r + 1] = e1;
    }
    if (payload == nullptr) return;
    const int64_t bit0 = (int64_t)r * rec_bits;
    if ((rec_bits & 7) == 0) {                     // whole bytes: plain stores
        uint8_t* dst = payload + (bit0 >> 3);
        for (int i = 0; i < rec_bits / 8; ++i) dst[i] = (uint8_t)(v >> (rec_bits - 8 * (i + 1)));
        return;
    }
    // straddling records: the record's bits, MSB-first from bit0, OR-ed into
    // the little-endian 32-bit words that hold those bytes
    const int sh = (int)(bit0 & 7);
    const int nbytes = (sh + rec_bits + 7) >> 3;   // <= 9
    const uint64_t top = v << (64 - rec_bits);     // record at the MSB of a 64-bit window
    uint32_t* words = reinterpret_cast<uint32_t*>(payload);
    for (int i = 0; i < nbytes; ++i) {
        // bits [8 i - sh, 8 i - sh + 8) of the record go to byte byte0 + i
        const int lo = 8 * i - sh;
        uint32_t byte;
        if (lo < 0) byte = (uint32_t)(top >> (64 - 8 + sh)) & (0xffu >> sh);
        else if (lo < 64) byte = (uint32_t)((top << lo) >> 56);
        else byte = 0u;
        if (byte == 0u) continue;
        const int64_t j = (bit0 >> 3) + i;
        atomicOr(&words[j >> 2], byte << (8 * (j & 3)));
    }
}

// NEXT-2 K-means (Lloyd) step for the RVQ codebooks: assignment with the
// encoder's fp32 distance and tie rule, then per-cluster sums in 2^-40 fixed
// point (int64: integer addition is associative, so the sums -- and the
// centroids -- do not depend on thread order).  Block partials in shared
// memory, one global atomic per (block, cluster, field).
constexpr double kFix = 1099511627776.0;   // 2^40

__global__ void __launch_bounds__(256) kmeans_assign_kernel(const float* __restrict__ pts, int n,
                                                            int B, const float* __restrict__ cent,
                                                            uint32_t* __restrict__ assign,
                                                            unsigned long long* __restrict__ acc) {
    __shared__ float sc[256 * 3];
    __shared__ unsigned long long sa[256 * 4];
    for (int i = threadIdx.x; i < B * 3; i += blockDim.x) sc[i] = cent[i];
    for (int i = threadIdx.x; i < B * 4; i += blockDim.x) sa[i] = 0ull;
    __syncthreads();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        const float x0 = pts[3 * (size_t)i], x1 = pts[3 * (size_t)i + 1], x2 = pts[3 * (size_t)i + 2];
        int best = 0;
        float bestd = __int_as_float(0x7f800000);
        for (int k = 0; k < B; ++k) {
            const float d0 = __fsub_rn(sc[3 * k], x0), d1 = __fsub_rn(sc[3 * k + 1], x1);
            const float d2 = __fsub_rn(sc[3 * k + 2], x2);
            float dd = __fmul_rn(d0, d0);
            dd = __fadd_rn(dd, __fmul_rn(d1, d1));
            dd = __fadd_rn(dd, __fmul_rn(d2, d2));
            if (dd < bestd) {
                bestd = dd;
                best = k;
            }
        }
        if (assign != nullptr) assign[i] = (uint32_t)best;
        uint32_t* a = reinterpret_cast<uint32_t*>(sa) + 8 * best;   // (lo, hi) pairs
        shared_add_u64(a + 0, (unsigned long long)__double2ll_rn((double)x0 * kFix));
        shared_add_u64(a + 2, (unsigned long long)__double2ll_rn((double)x1 * kFix));
        shared_add_u64(a + 4, (unsigned long long)__double2ll_rn((double)x2 * kFix));
        atomicAdd(a + 6, 1u);
    }
    __syncthreads();
    const uint32_t* sp = reinterpret_cast<const uint32_t*>(sa);
    for (int k = threadIdx.x; k < B; k += blockDim.x)
        if (shared_read_u64(sp + 8 * k + 6) != 0ull)
            for (int j = 0; j < 4; ++j) atomicAdd(&acc[4 * k + j], shared_read_u64(sp + 8 * k + 2 * j));
}

// New centroids (empty clusters keep theirs, reading R31); re-zeroes acc.
__global__ void kmeans_update_kernel(int B, float* __restrict__ cent,
                                     unsigned long long* __restrict__ acc) {
    for (int k = threadIdx.x; k < B; k += blockDim.x) {
        const long long c = (long long)acc[4 * k + 3];
        if (c > 0)
            for (int j = 0; j < 3; ++j)
                cent[3 * k + j] =
                    (float)((double)(long long)acc[4 * k + j] * (1.0 / kFix) / (double)c);
        for (int j = 0; j < 4; ++j) acc[4 * k + j] = 0ull;
    }
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

cudaError_t launch_vq_encode(const float* params, bool logit, const gi_codec_meta& meta,
                             uint8_t* payload, float* eff, cudaStream_t s) {
    if (meta.n == 0) return cudaSuccess;
    int ib = 1;
    while ((1 << ib) < meta.codebook) ++ib;
    const int rec = 32 + 3 * meta.bits + meta.stages * ib;
    if (payload != nullptr && (rec & 7) != 0) {
        const size_t bytes = ((size_t)rec * meta.n + 7) / 8;
        // whole 32-bit words (the atomics OR into words); the caller's buffer
        // is rounded the same way by gi_vq_encode's size check
        cudaError_t e = cudaMemsetAsync(payload, 0, (bytes + 3) & ~(size_t)3, s);
        if (e != cudaSuccess) return e;
    }
    vq_encode_kernel<<<(meta.n + 255) / 256, 256, 0, s>>>(
        reinterpret_cast<const float4*>(params), meta.n, logit, meta.bits, meta.stages,
        meta.codebook, ib, rec, meta.gamma[0], meta.gamma[1], meta.gamma[2], meta.beta[0],
        meta.beta[1], meta.beta[2], meta.codebooks, payload, reinterpret_cast<float4*>(eff));
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_kmeans_step(const float* points, int n, int B, float* centroids,
                               uint32_t* assign, void* ws, cudaStream_t s) {
    auto* acc = static_cast<unsigned long long*>(ws);
    if (n > 0) {
        kmeans_assign_kernel<<<(n + 255) / 256, 256, 0, s>>>(points, n, B, centroids, assign, acc);
        note_launches(1);
    }
    kmeans_update_kernel<<<1, 256, 0, s>>>(B, centroids, acc);
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace gi
