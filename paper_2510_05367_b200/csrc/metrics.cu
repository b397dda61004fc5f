// Per-frame PSNR / SSIM of two b=1 videos on the GPU (§8 f4): the quality
// columns of compare / ablate / sweep-n / export-plots
// (proj/src/pipeline.cpp:278-376) at config-C scale, where the reference's
// scalar double loops (proj/src/metrics.cpp:10-75) take minutes.
//
// Arithmetic follows the reference per element and per 7x7 window exactly
// (double sums in the loop order dy, dx; every product, sum and quotient an
// explicitly rounded double op, no FMA contraction), so each window's SSIM
// term is bit-identical; only the final sums over windows / pixels run as
// fixed-order block trees instead of one sequential loop (~1e-16 relative).
#include "metrics.cuh"

namespace lc {
namespace {

constexpr int kWin = 7;        // kSsimWindow (metrics.hpp:24)
constexpr double kCap = 99.0;  // kPsnrCap (metrics.hpp:17)
constexpr int kT = 16;         // SSIM output tile (16 x 16 windows per block)

__device__ double block_sum(double v, double* red) {
    // fixed-order tree over blockDim.x (power of two) values
    red[threadIdx.x] = v;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (static_cast<int>(threadIdx.x) < s) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + s]);
        __syncthreads();
    }
    return red[0];
}

// grid (nb, t): block x of frame y sums (a-b)^2 over its contiguous slice
__global__ void __launch_bounds__(256) sqdiff_kernel(const float* a, const float* b, int64_t fr, int64_t per,
                                                     double* partial) {
    __shared__ double red[256];
    const int64_t f0 = static_cast<int64_t>(blockIdx.y) * fr;
    const int64_t i0 = static_cast<int64_t>(blockIdx.x) * per;
    const int64_t i1 = i0 + per < fr ? i0 + per : fr;
    double acc = 0.0;
    for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        const double d = __dsub_rn(static_cast<double>(a[f0 + i]), static_cast<double>(b[f0 + i]));
        acc = __dadd_rn(acc, __dmul_rn(d, d));
    }
    const double s = block_sum(acc, red);
    if (threadIdx.x == 0) partial[static_cast<size_t>(blockIdx.y) * gridDim.x + blockIdx.x] = s;
}

// grid (tiles_x, tiles_y, t*c): 16x16 windows of one plane per block
__global__ void __launch_bounds__(256) ssim_kernel(const float* a, const float* b, int h, int w, double c1,
                                                   double c2, double* partial) {
    __shared__ float sa_t[kT + kWin - 1][kT + kWin - 1];
    __shared__ float sb_t[kT + kWin - 1][kT + kWin - 1];
    __shared__ double red[256];
    const int64_t plane = static_cast<int64_t>(blockIdx.z) * h * w;
    const int x0 = blockIdx.x * kT, y0 = blockIdx.y * kT;
    constexpr int E = kT + kWin - 1;
    for (int i = threadIdx.x; i < E * E; i += blockDim.x) {
        const int yy = y0 + i / E, xx = x0 + i % E;
        const bool in = yy < h && xx < w;
        sa_t[i / E][i % E] = in ? a[plane + static_cast<int64_t>(yy) * w + xx] : 0.f;
        sb_t[i / E][i % E] = in ? b[plane + static_cast<int64_t>(yy) * w + xx] : 0.f;
    }
    __syncthreads();
    const int tx = threadIdx.x % kT, ty = threadIdx.x / kT;
    double v = 0.0;
    if (x0 + tx + kWin <= w && y0 + ty + kWin <= h) {
        double sa = 0, sb = 0, saa = 0, sbb = 0, sab = 0;
        for (int dy = 0; dy < kWin; ++dy)
            for (int dx = 0; dx < kWin; ++dx) {
                const double va = sa_t[ty + dy][tx + dx], vb = sb_t[ty + dy][tx + dx];
                sa = __dadd_rn(sa, va);
                sb = __dadd_rn(sb, vb);
                saa = __dadd_rn(saa, __dmul_rn(va, va));
                sbb = __dadd_rn(sbb, __dmul_rn(vb, vb));
                sab = __dadd_rn(sab, __dmul_rn(va, vb));
            }
        const double inv_n = 1.0 / static_cast<double>(kWin * kWin);
        const double mu_a = __dmul_rn(sa, inv_n), mu_b = __dmul_rn(sb, inv_n);
        const double var_a = __dsub_rn(__dmul_rn(saa, inv_n), __dmul_rn(mu_a, mu_a));
        const double var_b = __dsub_rn(__dmul_rn(sbb, inv_n), __dmul_rn(mu_b, mu_b));
        const double cov = __dsub_rn(__dmul_rn(sab, inv_n), __dmul_rn(mu_a, mu_b));
        const double num = __dmul_rn(__dadd_rn(__dmul_rn(__dmul_rn(2.0, mu_a), mu_b), c1),
                                     __dadd_rn(__dmul_rn(2.0, cov), c2));
        const double den = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(mu_a, mu_a), __dmul_rn(mu_b, mu_b)), c1),
                                     __dadd_rn(__dadd_rn(var_a, var_b), c2));
        v = __ddiv_rn(num, den);
    }
    const double s = block_sum(v, red);
    if (threadIdx.x == 0)
        partial[(static_cast<size_t>(blockIdx.z) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = s;
}

}  // namespace

cudaError_t video_metrics(const float* a, const float* b, int64_t t, int64_t c, int64_t h, int64_t w,
                          double data_range, double* psnr, double* ssim, cudaStream_t st) {
    const int64_t fr = c * h * w;
    // PSNR: per-frame sum of squared differences
    const int nb = static_cast<int>(std::min<int64_t>(1024, (fr + 65535) / 65536));
    const int64_t per = (fr + nb - 1) / nb;
    const int tx = static_cast<int>((w + kT - 1) / kT), ty = static_cast<int>((h + kT - 1) / kT);
    const size_t n_ps = static_cast<size_t>(t) * nb, n_ss = static_cast<size_t>(t * c) * tx * ty;
    double* dp = nullptr;
    cudaError_t e = cudaMallocAsync(&dp, (n_ps + n_ss) * sizeof(double), st);
    if (e != cudaSuccess) return e;
    sqdiff_kernel<<<dim3(nb, static_cast<unsigned>(t)), 256, 0, st>>>(a, b, fr, per, dp);
    const double c1 = (0.01 * data_range) * (0.01 * data_range);
    const double c2 = (0.03 * data_range) * (0.03 * data_range);
    ssim_kernel<<<dim3(tx, ty, static_cast<unsigned>(t * c)), 256, 0, st>>>(a, b, static_cast<int>(h),
                                                                            static_cast<int>(w), c1, c2, dp + n_ps);
    e = cudaGetLastError();
    std::vector<double> hp(n_ps + n_ss);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hp.data(), dp, hp.size() * sizeof(double), cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(dp, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    const double windows = static_cast<double>(c) * static_cast<double>(h - kWin + 1) * static_cast<double>(w - kWin + 1);
    for (int64_t f = 0; f < t; ++f) {
        double sq = 0.0;
        for (int i = 0; i < nb; ++i) sq += hp[static_cast<size_t>(f) * nb + i];
        const double mse = sq / static_cast<double>(fr);
        psnr[f] = mse == 0.0 ? kCap : std::min(kCap, 10.0 * std::log10(data_range * data_range / mse));
        double tot = 0.0;
        const size_t base = n_ps + static_cast<size_t>(f) * c * tx * ty;
        for (size_t i = 0; i < static_cast<size_t>(c) * tx * ty; ++i) tot += hp[base + i];
        ssim[f] = tot / windows;
    }
    return cudaSuccess;
}

}  // namespace lc
