// K8: fused tap-to-N convolutions with a tiny output channel count, the
// U-Net head (3x3 conv c_in -> C <= 4, conditioning affine, bias;
// unet.cpp:76-97 run_conv_block for "head") and the decoder's last stage
// (nearest 2x upsample + 3x3 conv + bias; codec.cpp:96-124, tensor.cpp:
// 160-196, :232-248).  One persistent tcgen05 kernel: a TMA-staged window of
// pixels with a one-pixel halo times the tap bank (N = taps x C columns:
// for the head the 9 taps of the 3x3 kernel, engine.cu tap_bank; for the
// decoder every (output parity, 2x2 source tap) pair's merged weights,
// engine.cu subpix_tap_bank) into TMEM; then each output pixel sums its taps
// from shared memory and is stored straight into the fp32 planar output.
// Replaces the tap-to-N conv + tap/subpix gather kernel pairs: no fp32
// intermediate in HBM.
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace lc {

enum TapMode : int {
    kTapSubpix = 0,  // decoder: 4 output parities x 2x2 taps, output (n, C, 2H, 2W)
    kTapConv3 = 1,   // head: 3x3 taps, output (n, C, H, W), scale/offset affine
};

struct TapTcParams {
    CUtensorMap tmA;      // input (cs, W, H, n) fp16, box (64, kTapSX, kTapSY, 1), SW128
    const __half* w;      // [N][kb*64] fp16, row t*C + c (head) or (p*4+t)*C + c (decoder)
    const float* bias;    // [C]
    const float* wsum;    // head: [9][C] per-tap weight sums (offset correction)
    float scale;          // y = scale * acc (head: s / wscale; decoder: 1 / wscale)
    float shift;          // head: conditioning offset o
    float* out;           // planar fp32
    int n, H, W, C, N, kb;
    Window win;           // head: v* zero-padding window, o* output window (engine.hpp)
    int tiles_x, tiles_y, num_tiles;
    // head only, pair_T > 0: the sampler step fused into the epilogue
    // (cfg_combine + reverse_step_*, sampler.cpp:95-133, the rounding order
    // of kernels.cu step_kernel).  Images n and n + pair_T are the uncond /
    // cond branches (pipeline.cpp:127-131); a CTA runs the two tiles of one
    // (frame, tile) pair back to back, keeps e_u in shared memory and writes
    //   x_out = a*x + b*((1-g)*e_u + g*e_c)  [+ c*z]
    // instead of eps (which never reaches HBM); non-finite results raise
    // *bad (the next step's check_input, unet.cpp:134).
    int cfast;  // epilogue task order: 1 channel fastest (set at launch, LC_TAP_CFAST)
    int pair_T;
    const float* x;
    float* x_out;
    const float* z;  // nullable: ancestral noise
    float g, a, b, c;
    int* bad;
};

// Core tile kTapTX x TY pixels; the staged window adds a one-pixel halo on
// every side (TMA box kTapSX x (TY + 2)).  TY = tap_tile_rows(...): the head
// 5; the decoder 4 (a 3-stage A ring) where it fits, else 5 (2 stages).
constexpr int kTapTX = 64, kTapSX = kTapTX + 2;
int tap_tile_rows(int mode, int C, int kb, int N);
constexpr int kTapMaxKb = 5;  // c_in <= 320

cudaError_t launch_tap_tc(int mode, const TapTcParams& p, cudaStream_t st);
// Whether launch_tap_tc accepts this geometry (output channels, K blocks,
// tap columns; shared-memory fit).
bool tap_tc_supported(int mode, int C, int kb, int N);

}  // namespace lc
