// a4. L2 loss + analytic backward (Appendix A).
//
// Fused per-tile kernel: pass 1 recomputes C (Eq. 7) for the tile's pixels,
// forms g = dL/dC = 2 (C - T) / (3HW) in registers and a per-tile partial of
// the squared error; pass 2 walks the same key list and, for every pair
// (n, pixel) with the pixel in n's box, accumulates
//     dc'_n      += g w                                   (A.1)
//     gamma       = dL/dsigma = -w <g, c'_n>              (A.1, R12)
//     S_u += gamma u, S_v += gamma v, S_uu += gamma u^2, S_uv += gamma u v,
//     S_vv += gamma v^2      with (u, v) = kappa L^-1 d,  sigma = (u^2+v^2)/(2 kappa^2)
// i.e. the 5 moments from which dsigma/dmu (sign R13) and
// dsigma/dSigma = -1/2 Sigma^-1 d d^T Sigma^-1 chained through
// Sigma = L L^T (A.2, R14) follow in closed form per Gaussian.
// The 8 values are reduced over the warp by a transpose-reduce (9 SHFL),
// over the 8 warps of the tile in shared memory in a FIXED order, and
// written once per (tile, Gaussian) to the key's pre-sort slot
// gauss_offset[gid] + rank-of-tile-in-rect: no atomics, deterministic.
// finalize_kernel then sums each Gaussian's contiguous slots in order and
// applies the per-Gaussian chain rule (and tanh, App. C).
#include "raster_common.cuh"

namespace gi {
namespace {

constexpr int kSub = 32;   // Gaussians per reduction sub-batch

struct BwdShared {
    StagedRecords sr;
    uint32_t slot[256];                 // pre-sort key slot of each staged record
    float red[kWarps][kSub][8];         // per-warp reduced partials
    float sse[kWarps];
};

// Transpose-reduce 8 per-lane values over the warp: after it, lane l with
// (l & 3) == 0 holds the warp sum of value index (l >> 2).
__device__ __forceinline__ float warp_reduce8(float v0, float v1, float v2, float v3, float v4,
                                              float v5, float v6, float v7, int lane) {
    const bool h4 = lane & 16;
    float k0 = h4 ? v4 : v0, k1 = h4 ? v5 : v1, k2 = h4 ? v6 : v2, k3 = h4 ? v7 : v3;
    const float s0 = h4 ? v0 : v4, s1 = h4 ? v1 : v5, s2 = h4 ? v2 : v6, s3 = h4 ? v3 : v7;
    k0 += __shfl_xor_sync(kFull, s0, 16);
    k1 += __shfl_xor_sync(kFull, s1, 16);
    k2 += __shfl_xor_sync(kFull, s2, 16);
    k3 += __shfl_xor_sync(kFull, s3, 16);
    const bool h3 = lane & 8;
    float j0 = h3 ? k2 : k0, j1 = h3 ? k3 : k1;
    const float t0 = h3 ? k0 : k2, t1 = h3 ? k1 : k3;
    j0 += __shfl_xor_sync(kFull, t0, 8);
    j1 += __shfl_xor_sync(kFull, t1, 8);
    const bool h2 = lane & 4;
    float i0 = h2 ? j1 : j0;
    const float r0 = h2 ? j0 : j1;
    i0 += __shfl_xor_sync(kFull, r0, 4);
    i0 += __shfl_xor_sync(kFull, i0, 2);
    i0 += __shfl_xor_sync(kFull, i0, 1);
    return i0;
}

__global__ void __launch_bounds__(256) backward_tile_kernel(
    const Proj* __restrict__ proj, const uint32_t* __restrict__ key_gid,
    const uint32_t* __restrict__ tile_range, const uint32_t* __restrict__ gauss_offset, int W,
    int H, int T, int TX, const float* __restrict__ dL_dimage, const float* __restrict__ target,
    float norm, int64_t cap, float* __restrict__ partial, float* __restrict__ sse_part,
    float* __restrict__ image_out) {
    __shared__ BwdShared sh;
    const TileCtx t = make_tile_ctx(W, H, TX);
    const uint32_t s = tile_range[t.img * T + t.tile];
    const uint32_t e = tile_range[t.img * T + t.tile + 1];
    const size_t P = (size_t)W * H;
    const size_t pix = (size_t)t.img * 3 * P + (size_t)t.y * W + t.x;
    bool staged_all = false;   // pass 1 left the whole list in shared memory

    float g0 = 0.f, g1 = 0.f, g2 = 0.f;
    if (dL_dimage != nullptr) {
        if (t.in_image) {
            g0 = dL_dimage[pix];
            g1 = dL_dimage[pix + P];
            g2 = dL_dimage[pix + 2 * P];
        }
    } else {
        // ---- pass 1: forward (Eq. 7) ----
        float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f;
        for (uint32_t base = s; base < e; base += 256) {
            const int cnt = (int)min(256u, e - base);
            __syncthreads();
            stage_record(sh.sr, proj, key_gid, base, cnt, t, nullptr);
            __syncthreads();
#pragma unroll 1
            for (int q = 0; q < cnt; q += 32) {
                const int jl = q + t.lane;
                const bool ov = jl < cnt && warp_overlaps(sh.sr.c[jl], t);
                unsigned m = __ballot_sync(kFull, ov);
                while (m) {
                    const int j = q + __ffs(m) - 1;
                    m &= m - 1;
                    const float4 A = sh.sr.a[j];
                    const float4 B = sh.sr.b[j];
                    const PairEval pe = eval_pair(A, B, t);
                    const float w = pixel_in_box(sh.sr.c[j], t) ? pe.w : 0.f;
                    acc0 = fmaf(B.y, w, acc0);
                    acc1 = fmaf(B.z, w, acc1);
                    acc2 = fmaf(B.w, w, acc2);
                }
            }
        }
        staged_all = (e - s) <= 256u;
        float sq = 0.f;
        if (t.in_image) {
            const float r0 = acc0 - target[pix];
            const float r1 = acc1 - target[pix + P];
            const float r2 = acc2 - target[pix + 2 * P];
            g0 = norm * r0;
            g1 = norm * r1;
            g2 = norm * r2;
            sq = fmaf(r0, r0, fmaf(r1, r1, r2 * r2));
            if (image_out != nullptr) {
                image_out[pix] = acc0;
                image_out[pix + P] = acc1;
                image_out[pix + 2 * P] = acc2;
            }
        }
        if (sse_part != nullptr) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(kFull, sq, o);
            if (t.lane == 0) sh.sse[t.warp] = sq;
            __syncthreads();
            if (threadIdx.x == 0) {
                float tot = 0.f;
#pragma unroll
                for (int w = 0; w < kWarps; ++w) tot += sh.sse[w];
                sse_part[t.img * T + t.tile] = tot;
            }
        }
    }

    // ---- pass 2: gradients ----
    for (uint32_t base = s; base < e; base += 256) {
        const int cnt = (int)min(256u, e - base);
        __syncthreads();
        {
            const int j = threadIdx.x;
            if (!staged_all) stage_record(sh.sr, proj, key_gid, base, cnt, t, nullptr);
            if (j < cnt) {
                // slot of key (tile, gid) in the pre-sort (gid-major, row-major
                // rectangle) order; record j was staged by this same thread
                const uint32_t gid = key_gid[base + j];
                const int4 b = sh.sr.c[j];
                const int tx0 = b.x / kTile, tx1 = (b.x + b.y) / kTile, ty0 = b.z / kTile;
                sh.slot[j] = gauss_offset[gid] + (uint32_t)((t.ty - ty0) * (tx1 - tx0 + 1) + (t.tx - tx0));
            }
        }
        __syncthreads();
        for (int q = 0; q < cnt; q += kSub) {
            // zero this warp's reduction rows
            {
                float4* row = reinterpret_cast<float4*>(&sh.red[t.warp][t.lane][0]);
                row[0] = make_float4(0.f, 0.f, 0.f, 0.f);
                row[1] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
            const int jl = q + t.lane;
            const bool ov = jl < cnt && warp_overlaps(sh.sr.c[jl], t);
            unsigned m = __ballot_sync(kFull, ov);
            __syncwarp();
            while (m) {
                const int jj = __ffs(m) - 1;
                m &= m - 1;
                const int j = q + jj;
                const float4 A = sh.sr.a[j];
                const float4 B = sh.sr.b[j];
                const PairEval pe = eval_pair(A, B, t);
                const float w = pixel_in_box(sh.sr.c[j], t) ? pe.w : 0.f;
                const float gw0 = g0 * w, gw1 = g1 * w, gw2 = g2 * w;
                // gamma = dL/dsigma = -w <g, c'>
                const float gam = -fmaf(B.y, gw0, fmaf(B.z, gw1, B.w * gw2));
                const float gu = gam * pe.u, gv = gam * pe.v;
                const float r = warp_reduce8(gw0, gw1, gw2, gu, gv, gu * pe.u, gu * pe.v,
                                             gv * pe.v, t.lane);
                if ((t.lane & 3) == 0) sh.red[t.warp][jj][t.lane >> 2] = r;
            }
            __syncthreads();
            {
                const int jj = threadIdx.x >> 3, c = threadIdx.x & 7;
                if (q + jj < cnt) {
                    float acc = 0.f;
#pragma unroll
                    for (int w = 0; w < kWarps; ++w) acc += sh.red[w][jj][c];
                    const uint32_t slot = sh.slot[q + jj];
                    if ((int64_t)slot < cap) partial[(size_t)slot * 8 + c] = acc;
                }
            }
            __syncthreads();
        }
    }
}

// Per Gaussian: sum its tiles' partials in slot order, then the closed-form
// chain rule.  With p = u / kappa, q = v / kappa (so sigma = (p^2 + q^2) / 2,
// p = dx / l1, q = (dy - l2 p) / l3):
//   dsigma/ddx = (p - q l2 / l3) / l1,  dsigma/ddy = q / l3,  d = pixel - mu
//   dsigma/dl1 = -p dsigma/ddx, dsigma/dl2 = -p q / l3, dsigma/dl3 = -q^2 / l3
// (equal to <dsigma/dSigma, dSigma/dl> of A.2 with the R14 correction).
__global__ void __launch_bounds__(256) finalize_kernel(const float4* __restrict__ params,
                                                       const uint32_t* __restrict__ gauss_offset,
                                                       int total, int W, int H, uint32_t flags,
                                                       int64_t cap, const float* __restrict__ partial,
                                                       float4* __restrict__ grads) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= total) return;
    const uint32_t o0 = gauss_offset[g], o1 = gauss_offset[g + 1];
    float S[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (uint32_t o = o0; o < o1 && (int64_t)o < cap; ++o) {
        const float4 a = reinterpret_cast<const float4*>(partial)[2 * (size_t)o];
        const float4 b = reinterpret_cast<const float4*>(partial)[2 * (size_t)o + 1];
        S[0] += a.x; S[1] += a.y; S[2] += a.z; S[3] += a.w;
        S[4] += b.x; S[5] += b.y; S[6] += b.z; S[7] += b.w;
    }
    const float4 p0 = params[2 * (size_t)g], p1 = params[2 * (size_t)g + 1];
    float4 r0 = make_float4(0.f, 0.f, 0.f, 0.f), r1 = r0;
    if (o1 > o0) {
        const double l1 = (double)p0.z + 0.5, l2 = (double)p0.w, l3 = (double)p1.x + 0.5;
        const double ik = 1.0 / kKappa, ik2 = ik * ik;
        const double Sp = S[3] * ik, Sq = S[4] * ik;
        const double Spp = S[5] * ik2, Spq = S[6] * ik2, Sqq = S[7] * ik2;
        const double Ax = (Sp - Sq * l2 / l3) / l1;   // sum gamma dsigma/ddx
        const double Ay = Sq / l3;
        double sx = (double)W * 0.5, sy = (double)H * 0.5;
        if (flags == GI_POS_LOGIT) {
            const double chx = cosh((double)p0.x), chy = cosh((double)p0.y);
            sx /= chx * chx;
            sy /= chy * chy;
        }
        r0.x = (float)(-Ax * sx);                        // dmu = -dsigma/dd (R13)
        r0.y = (float)(-Ay * sy);
        r0.z = (float)(-(Spp - Spq * l2 / l3) / l1);     // dl1
        r0.w = (float)(-Spq / l3);                       // dl2
        r1.x = (float)(-Sqq / l3);                       // dl3
        r1.y = S[0];                                     // dc'
        r1.z = S[1];
        r1.w = S[2];
    }
    grads[2 * (size_t)g] = r0;
    grads[2 * (size_t)g + 1] = r1;
}

__global__ void __launch_bounds__(256) loss_kernel(const float* __restrict__ sse_part, int T,
                                                   double inv_count, float* __restrict__ loss) {
    __shared__ double sm[256];
    const int img = blockIdx.x;
    double acc = 0.0;
    for (int i = threadIdx.x; i < T; i += blockDim.x) acc += (double)sse_part[img * T + i];
    sm[threadIdx.x] = acc;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) sm[threadIdx.x] += sm[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) loss[img] = (float)(sm[0] * inv_count);
}

struct BwdWs {
    float* partial;
    float* sse;
    size_t bytes;
};

BwdWs carve(void* base, int n, int64_t cap, const gi_frame& f) {
    (void)n;
    const int T = tiles_x(f.width) * tiles_y(f.height);
    char* p = static_cast<char*>(base);
    BwdWs w;
    size_t off = 0;
    w.partial = reinterpret_cast<float*>(p + off); off += align_up(sizeof(float) * 8 * (size_t)cap);
    w.sse = reinterpret_cast<float*>(p + off); off += align_up(sizeof(float) * (size_t)T * f.batch);
    w.bytes = off;
    return w;
}

}  // namespace

size_t backward_ws_bytes(int n, int64_t cap, const gi_frame& f) { return carve(nullptr, n, cap, f).bytes; }

cudaError_t launch_backward_tiles(const Proj* proj, const uint32_t* key_gid,
                                  const uint32_t* tile_range, const uint32_t* gauss_offset, int n,
                                  const gi_frame& f, const float* dL_dimage, const float* target,
                                  int64_t cap, void* ws, float* image_out, cudaStream_t s) {
    (void)n;
    BwdWs w = carve(ws, n, cap, f);
    const int TX = tiles_x(f.width), T = TX * tiles_y(f.height);
    const double count = 3.0 * (double)f.width * (double)f.height;
    const float norm = (float)(2.0 / count);
    const bool mse = dL_dimage == nullptr;
    dim3 grid(T, f.batch);
    backward_tile_kernel<<<grid, 256, 0, s>>>(proj, key_gid, tile_range, gauss_offset, f.width,
                                              f.height, T, TX, dL_dimage, target, norm, cap,
                                              w.partial, mse ? w.sse : nullptr,
                                              mse ? image_out : nullptr);
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_backward_finalize(const float* params, const uint32_t* gauss_offset, int n,
                                     const gi_frame& f, uint32_t flags, bool mse, int64_t cap,
                                     void* ws, float* grads, float* loss, cudaStream_t s) {
    BwdWs w = carve(ws, n, cap, f);
    const int T = tiles_x(f.width) * tiles_y(f.height);
    const double count = 3.0 * (double)f.width * (double)f.height;
    const int total = n * f.batch;
    cudaError_t e = cudaSuccess;
    if (total > 0) {
        finalize_kernel<<<(total + 255) / 256, 256, 0, s>>>(
            reinterpret_cast<const float4*>(params), gauss_offset, total, f.width, f.height, flags,
            cap, w.partial, reinterpret_cast<float4*>(grads));
        note_launches(1);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    if (mse && loss != nullptr) {
        loss_kernel<<<f.batch, 256, 0, s>>>(w.sse, T, 1.0 / count, loss);
        note_launches(1);
        e = cudaGetLastError();
    }
    return e;
}

cudaError_t launch_backward(const float* params, const Proj* proj, const uint32_t* key_gid,
                            const uint32_t* tile_range, const uint32_t* gauss_offset, int n,
                            const gi_frame& f, uint32_t flags, const float* dL_dimage,
                            const float* target, int64_t cap, void* ws, float* grads, float* loss,
                            float* image_out, cudaStream_t s) {
    cudaError_t e = launch_backward_tiles(proj, key_gid, tile_range, gauss_offset, n, f, dL_dimage,
                                          target, cap, ws, image_out, s);
    if (e != cudaSuccess) return e;
    return launch_backward_finalize(params, gauss_offset, n, f, flags, dL_dimage == nullptr, cap,
                                    ws, grads, loss, s);
}

}  // namespace gi
