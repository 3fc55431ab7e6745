// PSNR per image (harness metric, not on the hot path):
// 10 log10(1 / MSE) on values clamped to [0, 1], capped at 100 dB.
// Two launches: per-block fp64 partial sums (fixed grid, fixed order), then
// one block per image.  The per-image values are what the multi-GPU driver
// all-gathers over NCCL.
#include "gi_internal.cuh"

namespace gi {
namespace {

constexpr int kPsnrBlocks = 148 * 2;

__global__ void __launch_bounds__(256) psnr_partial_kernel(const float* __restrict__ image,
                                                           const float* __restrict__ target,
                                                           int64_t count, double* __restrict__ part) {
    __shared__ double sm[256];
    const int img = blockIdx.y;
    const float* a = image + (size_t)img * count;
    const float* b = target + (size_t)img * count;
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float x = fminf(fmaxf(a[i], 0.f), 1.f);
        const float y = fminf(fmaxf(b[i], 0.f), 1.f);
        const double d = (double)x - (double)y;
        acc += d * d;
    }
    sm[threadIdx.x] = acc;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) sm[threadIdx.x] += sm[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[(size_t)img * gridDim.x + blockIdx.x] = sm[0];
}

__global__ void __launch_bounds__(256) psnr_final_kernel(const double* __restrict__ part, int nparts,
                                                         int64_t count, float* __restrict__ psnr) {
    __shared__ double sm[256];
    const int img = blockIdx.x;
    double acc = 0.0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) acc += part[(size_t)img * nparts + i];
    sm[threadIdx.x] = acc;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) sm[threadIdx.x] += sm[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double mse = sm[0] / (double)count;
        psnr[img] = mse <= 1e-10 ? 100.0f : (float)fmin(100.0, 10.0 * log10(1.0 / mse));
    }
}

}  // namespace

cudaError_t launch_psnr(const float* image, const float* target, const gi_frame& f, float* psnr,
                        void* ws, cudaStream_t s) {
    const int64_t count = 3LL * f.width * f.height;
    double* part = static_cast<double*>(ws);
    dim3 grid(kPsnrBlocks, f.batch);
    psnr_partial_kernel<<<grid, 256, 0, s>>>(image, target, count, part);
    note_launches(1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    psnr_final_kernel<<<f.batch, 256, 0, s>>>(part, kPsnrBlocks, count, psnr);
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace gi
