// GPU per-frame PSNR / SSIM (metrics.cu).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

namespace lc {

// a, b: device pointers to two b=1 videos {t,c,h,w} fp32.  psnr/ssim: host
// arrays of t doubles.  Synchronises `st`.
cudaError_t video_metrics(const float* a, const float* b, int64_t t, int64_t c, int64_t h, int64_t w,
                          double data_range, double* psnr, double* ssim, cudaStream_t st);

}  // namespace lc
