// K8: the decoder's last stage -- nearest 2x upsample + 3x3 conv (c_in ->
// C <= 4 image channels) + bias, written straight into the fp32 planar video
// (codec.cpp:96-124 decode_batch's last block; tensor.cpp:160-196 conv2d,
// :232-248 upsample2).  One persistent tcgen05 kernel: a TMA-staged window of
// low-res pixels (with a one-pixel halo) times the 16*C-column tap bank
// (engine.cu subpix_tap_bank: every (output parity, 2x2 source tap) pair's
// merged 3x3 weights) into TMEM, then per output parity the four taps of
// each output pixel are summed from shared memory.  Replaces the tap-to-N
// conv + subpix_gather_kernel pair: no fp32 intermediate in HBM.
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace lc {

struct SubpixTcParams {
    CUtensorMap tmA;      // low-res activation (cs, W, H, n) fp16, box (64, kSX, kSY, 1), SW128
    const __half* w;      // [N = 16*C][kb*64] fp16, row (p*4+t)*C + c
    const float* bias;    // [C]
    float* out;           // planar (n, C, 2H, 2W) fp32
    int n, H, W, C, kb;   // low-res extents, image channels, 64-channel K blocks
    int tiles_x, tiles_y, num_tiles;
};

constexpr int kSubpixTX = 64, kSubpixTY = 5;                        // core tile (low-res pixels)
constexpr int kSubpixSX = kSubpixTX + 2, kSubpixSY = kSubpixTY + 2;  // staged window with halo

cudaError_t launch_subpix_tc(const SubpixTcParams& p, cudaStream_t st);

}  // namespace lc
