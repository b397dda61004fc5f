// HBM-bound and thin-channel kernels of the path (everything that is not a
// dense tensor-core contraction).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace lc {

// Valid (readable) window + output region of one tiled launch, in pixel
// coordinates of the operand.  Reads outside [vy0,vy1)x[vx0,vx1) are zero
// (the reference's crop-then-conv, proj/src/chunk.cpp:182-188).
struct Window {
    int vy0, vy1, vx0, vx1;  // valid input window
    int oy0, oy1, ox0, ox1;  // output region
};

// Thin-input conv (c_in <= 8): fp32 NCHW input -> fp16 NHWC output.
//  * stem of the denoiser (cfg_pair=1: writes both CFG branches; branch 1
//    reads x + 0.15f, proj/src/pipeline.cpp:127-131), conditioning affine
//    applied exactly as the reference (affine before zero padding);
//  * first decoder conv (cfg_pair=0, s=1, o=0 skips the affine).
// Arithmetic mirrors conv2d_window (tensor.cpp:170-193) in fp32.
struct ThinInArgs {
    const float* x;   // (nsrc, c_in, H, W)
    int nsrc, c_in, H, W;
    int cfg_pair;     // 1: output images = 2*nsrc
    float cond_bias;  // added to x for branch 1
    float s, o;
    int apply_affine;
    const float* w;   // [c_out][c_in][k][k]
    const float* bias;
    int c_out, k;
    int silu;
    __half* out;      // (nimg, H, W, cs_out)
    int cs_out;
    Window win;
};

// Patch gather for a thin-input conv run on the tensor cores: writes, per
// output pixel, the conditioned k*k*c_in input taps (zero for taps outside
// the valid window) as one fp16 row of `kp` channels (multiple of 64), so the
// conv becomes a 1x1 tensor-core GEMM with K = kp.  The conditioning uses the
// reference roundings (x [+0.15], then x*s+o).  Uses a.out/a.cs_out as the
// patch tensor (nimg, H, W, kp); weights/bias/silu fields are ignored.
cudaError_t launch_patch(const ThinInArgs& a, int kp, cudaStream_t st);

// Tap gather of a tap-to-N conv.  A thin-output k x k conv (c_out = C <= 4:
// the denoiser head) runs on the tensor cores as a 1x1 GEMM whose N axis is
// (tap, channel): y[t*C + c][px] = s * sum_ic w[c][ic][t] x[px][ic] (fp32,
// channel-planar [t*C + c][n][H][W]).  This kernel sums the in-window taps of each output pixel and adds
// the folded conditioning o * sum_{in-window t} wsum[t][c] + bias[c]
// (unet.cpp:78-97 run_conv_block: affine -> zero-padded conv), writing fp32
// NCHW.
struct TapGatherArgs {
    const float* y;
    int cs_y;
    int n, H, W, C, k;
    Window win;         // v*: materialised (zero-padding) window, o*: output window
    const float* wsum;  // [k*k][C]
    const float* bias;  // [C]
    float o;
    float* out;         // (n, C, H, W)
};
cudaError_t launch_tap_gather(const TapGatherArgs& a, cudaStream_t st);

// Sub-pixel tap gather of the last decoder conv (nearest 2x upsample + 3x3,
// codec.cpp:103-113): y[(p*4 + t)*C + c][n][H][W] (channel-planar) holds, per output parity
// p = (py, px) and merged 2x2 tap t = (dy, dx), the GEMM partial sums; the
// output pixel (2Y+py, 2X+px) is bias + the sum of its four in-range low-res
// neighbours (Y+dy-1+py, X+dx-1+px).  fp32 NCHW video (n, C, 2H, 2W).
struct SubpixGatherArgs {
    const float* y;
    int cs_y;
    int n, H, W, C;     // low-res extents
    const float* bias;  // [C]
    float* out;
};
cudaError_t launch_subpix_gather(const SubpixGatherArgs& a, cudaStream_t st);


// 2x2 mean pool 0.25f*(a+b+c+d) (tensor.cpp:206-225), fp16 NHWC.
cudaError_t launch_down2(const __half* in, __half* out, int nimg, int H, int W, int cs,
                         cudaStream_t st);
// Nearest 2x upsample (tensor.cpp:232-248), fp16 NHWC.
cudaError_t launch_up2(const __half* in, __half* out, int nimg, int H, int W, int cs,
                       cudaStream_t st);

// CFG combine + sampler update (sampler.cpp:95-133, pipeline.cpp:170-185):
//   eps = (1-g)*e_u + g*e_c ; x' = a*x + b*eps [; x' = 1*x' + c*z]
// with the reference's two-rounding order; raises *bad if x' is non-finite
// (the next step's check_input, unet.cpp:134).
struct StepArgs {
    const float* eps2;  // (2, n)
    const float* x;
    float* x_out;
    const float* z;     // nullable
    int64_t n;
    float g, a, b, c;
    int* bad;
};
cudaError_t launch_step(const StepArgs& a, cudaStream_t st);

// out = a*x + b*y with two roundings (linear, tensor.cpp:269-274); used for
// forward_noise (sampler.cpp:87-93).
cudaError_t launch_linear(float a, const float* x, float b, const float* y, float* out, int64_t n,
                          cudaStream_t st);

// Non-finite scan of a fp32 buffer (all_finite, tensor.cpp:376).
cudaError_t launch_isfinite(const float* x, int64_t n, int* bad, cudaStream_t st);

}  // namespace lc
