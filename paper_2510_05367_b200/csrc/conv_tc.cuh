// Implicit-GEMM convolution on tcgen05 tensor cores (sm_100a).
//
// Replaces the reference's scalar conv2d_window hot loop
// (proj/src/tensor.cpp:155-197), fused with the block prologue/epilogue of
// run_conv_block / run_up_block (proj/src/unet.cpp:78-122):
//   * the per-block conditioning affine x*s+o is folded algebraically:
//       conv(affine(x)) = s * conv_nobias(x) + o * sum_{in-bound taps} w + bias
//     so zero padding stays literal zeros exactly as in the reference;
//   * channel concat (up blocks) is a two-segment K loop, never materialised;
//   * nearest-upsample + conv3x3 runs "sub-pixel": per output parity class
//     the upsampled operand is a 2x2 conv over the low-res tensor with merged
//     taps, and the full-res skip operand is read with TMA element stride 2;
//   * bias, conditioning shift and SiLU run in the TMEM->register epilogue.
//
// GEMM view: M = output pixels (a TI x TH x TW spatial tile of <=128 pixels),
// N = output channels (BN <= 256 per CTA), K = segment x tap x channel in
// the weight rows; the MMAs accumulate in (segment, 64-channel block, tap)
// order, the order the halo staging (below) consumes its boxes in, so every
// staging variant of a layer produces bit-identical sums.
// Activations are fp16 NHWC ("channels-last"), channel stride a multiple of
// 64 so one K block is one 128-byte SW128 row per pixel.
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace lc {

constexpr int kMaxTaps = 225;  // odd kernels up to 15x15 (ConvParams stays well under the 32 KB parameter limit)

// One K segment: one source tensor read through one TMA descriptor.
struct ConvSegDev {
    int ntaps;  // taps of this segment
    int ncb;    // 64-channel blocks per tap
    int kbase;  // first K element of this segment in a weight row
    int mx, my; // source coordinate = lattice * m + offset
    int wx0, wy0;  // origin of the tensor map window in source coordinates
    int8_t ox[4][kMaxTaps];  // per parity class, per tap
    int8_t oy[4][kMaxTaps];
};

// n / d and n % d for 0 <= n < 2^31 with one multiply-high (round-up
// magic number, set on the host): the per-tile schedule math runs on every
// epilogue warp, and 32-bit integer division is ~20 instructions.
struct FastDiv {
    uint32_t d = 1, m = 0, s = 0;
    void init(uint32_t div) {
        d = div;
        s = 0;
        while ((1ull << s) < div) ++s;
        m = static_cast<uint32_t>((((1ull << 32) * ((1ull << s) - div)) / div) + 1);
        if (div == 1) m = 0;
    }
#ifdef __CUDACC__
    __device__ __forceinline__ int div(int n) const {
        return static_cast<int>((__umulhi(static_cast<uint32_t>(n), m) + static_cast<uint32_t>(n)) >> s);
    }
    __device__ __forceinline__ int mod(int n) const { return n - div(n) * static_cast<int>(d); }
#endif
};

struct alignas(64) ConvParams {
    CUtensorMap tmA[2];  // activations, per segment: dims {C, W, H, N}
    CUtensorMap tmB;     // weights: dims {K_total, N_pad, P}
    ConvSegDev seg[2];
    int nseg;
    int n_img;                    // images = b*t
    int ly0[4], ly1[4], lx0[4], lx1[4];  // output region in lattice coords, per parity class
    int TI, TH, TW;               // pixel tile
    int tiles_x, tiles_y, tiles_i;
    int BN;                       // N tile
    int n_pad;                    // weight rows per parity class
    int c_out, cs_out;            // real output channels, output channel stride
    int out_h, out_w;             // output image extents (pixels)
    int sy, sx;                   // lattice -> output pixel multiplier (1 or 2)
    int py[4], px[4];             // per parity output offset
    __half* out;
    float* out32;                 // non-null: fp32 NCHW (img, c_out, out_h, out_w) output instead
    int shuffle_c;                // >0 (with out32): depth-to-space, channel p*shuffle_c+o ->
                                  // pixel (2Y+p/2, 2X+p%2), channel o of a shuffle_c-channel image
    const float* bias;            // [n_pad]
    const float* corr;            // [P][ncls][n_pad]   sum of in-bound tap weights
    int rc;                       // class radius (lattice units)
    int cy0, cy1, cx0, cx1;       // class window (lattice units)
    float scale;                  // s / weight_scale
    float shift;                  // o
    int silu;
    int cg;                       // 1: one CTA per M=128 tile; 2: CTA pair, M=256 (cta_group::2)
    int nparity;                  // parity classes (grid z of the schedule): 1 or 4
    int m_fastest;                // tile order: 1 weight-stationary (M fastest), 0 activation-stationary
    int epi_rot;                  // epilogue column-group rotation per tile (set at launch)
    int planar32;                 // with nhwc32: channel-planar [channel][img][y][x] instead of NHWC
    int nhwc32;                   // with out32: raw fp32 NHWC (channel stride cs_out), value
                                  // = scale * acc, no offsets/activation (tap-to-N GEMMs whose
                                  // taps are summed by a gather kernel)
    // fp16 outputs through TMA tensor stores: per parity class, the output
    // lattice {C, X, Y, img} of that class (window-clipped, so the TMA unit
    // drops out-of-window rows); each epilogue warp stages 32 pixels x 16
    // channels in shared memory and stores them as one box
    int tma_out;
    CUtensorMap tmO[4];
    // weight-stationary schedule (CG = 1): the CTAs are split into one group
    // per (parity, N tile) slab; each CTA loads its slab's whole K x BN
    // weight panel into shared memory once and streams only activation
    // tiles (small-K, small-N layers whose per-tile weight re-reads would
    // otherwise make them L2-bandwidth bound)
    int b_res;
    // halo operand staging (b_res, one segment, one-row tiles of 128 pixels
    // at source scale 1): per 64-channel block ONE box of hh rows x hw
    // pixels covering every tap's shifted tile is loaded (origin hox/hoy per
    // parity), and each tap's MMA reads its 128 rows at a row offset of that
    // box (a start-address shift of the SW128 descriptor, 128 B per pixel)
    // instead of a box of its own: hh*hw instead of ntaps*128 pixel rows
    int halo;
    int hw, hh;
    int hox[4], hoy[4];
    FastDiv fd_units, fd_ntiles, fd_par, fd_tx, fd_ty;  // launch-side divisors of tile_coord
};
// passed by value as a __grid_constant__ kernel parameter (32 KB limit)
static_assert(sizeof(ConvParams) < 16384, "ConvParams too large for a kernel parameter");

// CTA-group choice for a launch (the weight tensor map's box depends on it:
// each CTA of a pair stages BN/2 weight rows).
int conv_tc_cta_group(int BN, int m_tiles, int n_tiles, int parities, int k_blocks);

struct ConvTcConfig {
    int stages;
    int tmem_cols;
    size_t smem_bytes;
};

// Host launcher (conv_tc.cu).
cudaError_t launch_conv_tc(const ConvParams& p, int parities, cudaStream_t stream);
size_t conv_tc_smem_bytes(const ConvParams& p);
// Whether a layer with p.halo set (and hw/hh filled in) can run halo-staged:
// one segment, single CTAs, weight-stationary with >= 2 halo stages.
bool conv_tc_halo_fits(const ConvParams& p, int parities);

}  // namespace lc
