// HBM-bound and thin-channel kernels; see kernels.cuh.
#include "kernels.cuh"
#include "pdl.cuh"

namespace lc {

namespace {


// ------------------------------------------------------------- thin input
// One thread per (output pixel, output channel); weights staged in shared
// memory as [c_in*k*k][c_out] so a warp (consecutive oc) reads consecutive
// banks.  Exact reference order: bias, then (ic, ky, kx) ascending with
// out-of-window taps skipped, separate multiply and add roundings.
__global__ void thin_in_kernel(const ThinInArgs a) {
    extern __shared__ float wsm[];
    const int kk = a.k * a.k;
    const int nw = a.c_out * a.c_in * kk;
    for (int i = threadIdx.x; i < nw; i += blockDim.x) {
        const int oc = i / (a.c_in * kk), rest = i % (a.c_in * kk);
        wsm[rest * a.c_out + oc] = a.w[i];
    }
    __syncthreads();
    const int oh = a.win.oy1 - a.win.oy0, ow = a.win.ox1 - a.win.ox0;
    const int nimg = a.cfg_pair ? 2 * a.nsrc : a.nsrc;
    const int64_t total = static_cast<int64_t>(nimg) * oh * ow * a.c_out;
    const int r = (a.k - 1) / 2;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int oc = static_cast<int>(idx % a.c_out);
        int64_t px = idx / a.c_out;
        const int ox = a.win.ox0 + static_cast<int>(px % ow);
        px /= ow;
        const int oy = a.win.oy0 + static_cast<int>(px % oh);
        const int n = static_cast<int>(px / oh);
        const int src = n % a.nsrc;
        const bool branch1 = a.cfg_pair && n >= a.nsrc;
        const float* xs = a.x + static_cast<int64_t>(src) * a.c_in * a.H * a.W;
        float acc = a.bias[oc];
        for (int ic = 0; ic < a.c_in; ++ic) {
            for (int ky = 0; ky < a.k; ++ky) {
                const int iy = oy + ky - r;
                if (iy < a.win.vy0 || iy >= a.win.vy1) continue;
                for (int kx = 0; kx < a.k; ++kx) {
                    const int ix = ox + kx - r;
                    if (ix < a.win.vx0 || ix >= a.win.vx1) continue;
                    float v = xs[(static_cast<int64_t>(ic) * a.H + iy) * a.W + ix];
                    if (branch1) v = __fadd_rn(v, a.cond_bias);
                    if (a.apply_affine) v = __fadd_rn(__fmul_rn(v, a.s), a.o);
                    acc = __fadd_rn(acc, __fmul_rn(wsm[((ic * a.k + ky) * a.k + kx) * a.c_out + oc], v));
                }
            }
        }
        if (a.silu) acc = acc / (1.0f + expf(-acc));
        a.out[((static_cast<int64_t>(n) * a.H + oy) * a.W + ox) * a.cs_out + oc] = __float2half_rn(acc);
    }
}

// Fast path (c_in*k*k <= MAXIN): one thread per output pixel.  The
// conditioned input patch is formed once in registers (same roundings as
// above), then output channels are produced 8 at a time against weights
// staged in shared memory as [tap][cpad8] (warp-broadcast 16-byte reads),
// stored as one 16-byte fp16 vector.  Per output channel the accumulation is
// still bias, then (ic, ky, kx) ascending with skipped out-of-window taps.
template <int MAXIN>
__global__ void __launch_bounds__(128) thin_in_fast_kernel(const ThinInArgs a, int cpad8) {
    extern __shared__ float wsm[];
    const int kk = a.k * a.k, KK = a.c_in * kk;
    for (int i = threadIdx.x; i < KK * cpad8; i += blockDim.x) {
        const int t = i / cpad8, oc = i % cpad8;
        wsm[i] = oc < a.c_out ? a.w[oc * KK + t] : 0.0f;
    }
    float* bsm = wsm + KK * cpad8;
    for (int i = threadIdx.x; i < cpad8; i += blockDim.x) bsm[i] = i < a.c_out ? a.bias[i] : 0.0f;
    __syncthreads();
    const int oh = a.win.oy1 - a.win.oy0, ow = a.win.ox1 - a.win.ox0;
    const int nimg = a.cfg_pair ? 2 * a.nsrc : a.nsrc;
    const int64_t total = static_cast<int64_t>(nimg) * oh * ow;
    const int r = (a.k - 1) / 2;
    const int cmax = cpad8 < a.cs_out ? cpad8 : a.cs_out;
    // 8 lanes per pixel: lane g produces channel chunks g, g+8, ... so one
    // warp store instruction writes 4 pixels x 128 contiguous bytes.
    for (int64_t item = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; item < total * 8;
         item += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int g = static_cast<int>(item & 7);
        const int64_t idx = item >> 3;
        const int ox = a.win.ox0 + static_cast<int>(idx % ow);
        const int oy = a.win.oy0 + static_cast<int>((idx / ow) % oh);
        const int n = static_cast<int>(idx / (static_cast<int64_t>(ow) * oh));
        const int src = n % a.nsrc;
        const bool branch1 = a.cfg_pair && n >= a.nsrc;
        const float* xs = a.x + static_cast<int64_t>(src) * a.c_in * a.H * a.W;
        float v[MAXIN];
        uint64_t live = 0;
#pragma unroll
        for (int t = 0; t < MAXIN; ++t) {
            v[t] = 0.0f;
            if (t < KK) {
                const int ic = t / kk, ky = (t % kk) / a.k, kx = t % a.k;
                const int iy = oy + ky - r, ix = ox + kx - r;
                if (iy >= a.win.vy0 && iy < a.win.vy1 && ix >= a.win.vx0 && ix < a.win.vx1) {
                    float x = xs[(static_cast<int64_t>(ic) * a.H + iy) * a.W + ix];
                    if (branch1) x = __fadd_rn(x, a.cond_bias);
                    if (a.apply_affine) x = __fadd_rn(__fmul_rn(x, a.s), a.o);
                    v[t] = x;
                    live |= 1ull << t;
                }
            }
        }
        __half* dst = a.out + ((static_cast<int64_t>(n) * a.H + oy) * a.W + ox) * a.cs_out;
        for (int oc0 = g * 8; oc0 < cmax; oc0 += 64) {
            float acc[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] = bsm[oc0 + j];
#pragma unroll
            for (int t = 0; t < MAXIN; ++t) {
                if (t < KK && ((live >> t) & 1)) {
                    const float4 w0 = *reinterpret_cast<const float4*>(wsm + t * cpad8 + oc0);
                    const float4 w1 = *reinterpret_cast<const float4*>(wsm + t * cpad8 + oc0 + 4);
                    acc[0] = __fadd_rn(acc[0], __fmul_rn(w0.x, v[t]));
                    acc[1] = __fadd_rn(acc[1], __fmul_rn(w0.y, v[t]));
                    acc[2] = __fadd_rn(acc[2], __fmul_rn(w0.z, v[t]));
                    acc[3] = __fadd_rn(acc[3], __fmul_rn(w0.w, v[t]));
                    acc[4] = __fadd_rn(acc[4], __fmul_rn(w1.x, v[t]));
                    acc[5] = __fadd_rn(acc[5], __fmul_rn(w1.y, v[t]));
                    acc[6] = __fadd_rn(acc[6], __fmul_rn(w1.z, v[t]));
                    acc[7] = __fadd_rn(acc[7], __fmul_rn(w1.w, v[t]));
                }
            }
            __align__(16) __half2 h[4];
#pragma unroll
            for (int j = 0; j < 8; j += 2) {
                float p = acc[j], q = acc[j + 1];
                if (a.silu) {
                    p = __fdividef(p, 1.0f + __expf(-p));
                    q = __fdividef(q, 1.0f + __expf(-q));
                }
                h[j / 2] = __floats2half2_rn(p, q);
            }
            *reinterpret_cast<uint4*>(dst + oc0) = *reinterpret_cast<const uint4*>(h);
        }
    }
}

// --------------------------------------------------------- patch gather
// One thread per (output pixel, 8-tap group): writes 16 bytes of the fp16
// patch row; groups past c_in*k*k are zero.
__global__ void patch_kernel(const ThinInArgs a, int kp) {
    pdl_wait();
    const int kk = a.k * a.k, KK = a.c_in * kk;
    const int oh = a.win.oy1 - a.win.oy0, ow = a.win.ox1 - a.win.ox0;
    const int nimg = a.cfg_pair ? 2 * a.nsrc : a.nsrc;
    const int groups = kp / 8;
    const int64_t total = static_cast<int64_t>(nimg) * oh * ow * groups;
    const int r = (a.k - 1) / 2;
    for (int64_t item = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; item < total;
         item += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int g = static_cast<int>(item % groups);
        const int64_t idx = item / groups;
        const int ox = a.win.ox0 + static_cast<int>(idx % ow);
        const int oy = a.win.oy0 + static_cast<int>((idx / ow) % oh);
        const int n = static_cast<int>(idx / (static_cast<int64_t>(ow) * oh));
        const int src = n % a.nsrc;
        const bool branch1 = a.cfg_pair && n >= a.nsrc;
        const float* xs = a.x + static_cast<int64_t>(src) * a.c_in * a.H * a.W;
        __align__(16) __half h[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int t = g * 8 + j;
            float v = 0.0f;
            if (t < KK) {
                const int ic = t / kk, ky = (t % kk) / a.k, kx = t % a.k;
                const int iy = oy + ky - r, ix = ox + kx - r;
                if (iy >= a.win.vy0 && iy < a.win.vy1 && ix >= a.win.vx0 && ix < a.win.vx1) {
                    v = xs[(static_cast<int64_t>(ic) * a.H + iy) * a.W + ix];
                    if (branch1) v = __fadd_rn(v, a.cond_bias);
                    if (a.apply_affine) v = __fadd_rn(__fmul_rn(v, a.s), a.o);
                }
            }
            h[j] = __float2half_rn(v);
        }
        *reinterpret_cast<uint4*>(a.out + ((static_cast<int64_t>(n) * a.H + oy) * a.W + ox) * kp + g * 8) =
            *reinterpret_cast<const uint4*>(h);
    }
}

// Fast path of the patch gather: 3x3 taps, kp == 64, c_in = CIN (<= 7).
// One thread per output pixel: the 3 x 3 x CIN neighbourhood (row / column
// validity computed once), conditioned with the reference roundings, written
// as one 128-byte fp16 patch row (taps past CIN*9 are zero).  Consecutive
// threads walk x, so every tap load is coalesced.
template <int CIN>
__global__ void __launch_bounds__(256) patch3_kernel(const ThinInArgs a) {
    pdl_wait();
    const int ow = a.win.ox1 - a.win.ox0, oh = a.win.oy1 - a.win.oy0;
    const int idx = static_cast<int>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int nimg = a.cfg_pair ? 2 * a.nsrc : a.nsrc;
    if (idx >= nimg * oh * ow) return;
    const int row = idx / ow;
    const int ox = a.win.ox0 + (idx - row * ow);
    const int n = row / oh;
    const int oy = a.win.oy0 + (row - n * oh);
    const int src = n % a.nsrc;
    const bool branch1 = a.cfg_pair && n >= a.nsrc;
    const size_t plane = static_cast<size_t>(a.H) * a.W;
    const float* xs = a.x + static_cast<size_t>(src) * CIN * plane;
    bool rv[3], cv[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        rv[d] = oy + d - 1 >= a.win.vy0 && oy + d - 1 < a.win.vy1;
        cv[d] = ox + d - 1 >= a.win.vx0 && ox + d - 1 < a.win.vx1;
    }
    float v[64];
#pragma unroll
    for (int t = 0; t < 64; ++t) v[t] = 0.0f;
#pragma unroll
    for (int ic = 0; ic < CIN; ++ic)
#pragma unroll
        for (int ky = 0; ky < 3; ++ky)
#pragma unroll
            for (int kx = 0; kx < 3; ++kx) {
                if (rv[ky] && cv[kx]) {
                    float x = __ldg(xs + ic * plane + static_cast<size_t>(oy + ky - 1) * a.W + (ox + kx - 1));
                    if (branch1) x = __fadd_rn(x, a.cond_bias);
                    if (a.apply_affine) x = __fadd_rn(__fmul_rn(x, a.s), a.o);
                    v[(ic * 3 + ky) * 3 + kx] = x;
                }
            }
    uint4* dst = reinterpret_cast<uint4*>(a.out + ((static_cast<size_t>(n) * a.H + oy) * a.W + ox) * 64);
#pragma unroll
    for (int g = 0; g < 8; ++g) {
        __align__(16) __half2 h[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) h[j] = __floats2half2_rn(v[8 * g + 2 * j], v[8 * g + 2 * j + 1]);
        dst[g] = *reinterpret_cast<const uint4*>(h);
    }
}

// ------------------------------------------------------- tap gathers
// One thread per output pixel; consecutive threads walk x, so each tap read
// is a 16 B (C = 4) load at a 16*k*k-float stride, served from L2 (y was
// just written by the GEMM).
template <int K>
__global__ void __launch_bounds__(256) tap_gather_kernel(const TapGatherArgs a) {
    pdl_wait();
    const int ow = a.win.ox1 - a.win.ox0, oh = a.win.oy1 - a.win.oy0;
    const int idx = static_cast<int>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int c = static_cast<int>(blockIdx.y);  // output channel
    if (idx >= a.n * oh * ow) return;
    const int row = idx / ow;
    const int x = a.win.ox0 + (idx - row * ow);
    const int n = row / oh;
    const int yy = a.win.oy0 + (row - n * oh);
    constexpr int r = K / 2;
    const size_t plane = static_cast<size_t>(a.n) * a.H * a.W;  // one (tap, channel) plane of y
    const float* base = a.y + static_cast<size_t>(c) * plane + static_cast<size_t>(n) * a.H * a.W;
    float acc = 0.f, ws = 0.f;
#pragma unroll
    for (int ky = 0; ky < K; ++ky) {
        const int sy = yy + ky - r;
        const bool rin = sy >= a.win.vy0 && sy < a.win.vy1;
#pragma unroll
        for (int kx = 0; kx < K; ++kx) {
            const int sx = x + kx - r;
            const bool in = rin && sx >= a.win.vx0 && sx < a.win.vx1;
            const int t = ky * K + kx;
            // every tap load issued (clamped address), out-of-window ones discarded
            const float v = __ldg(base + static_cast<size_t>(t * a.C) * plane + static_cast<size_t>(in ? sy : yy) * a.W +
                                  (in ? sx : x));
            acc += in ? v : 0.f;
            ws += in ? __ldg(a.wsum + t * a.C + c) : 0.f;
        }
    }
    a.out[(static_cast<size_t>(n) * a.C + c) * a.H * a.W + static_cast<size_t>(yy) * a.W + x] =
        acc + fmaf(a.o, ws, __ldg(a.bias + c));
}

// One thread per (low-res pixel, output parity): its output pixel x C
// channels.  y is channel-planar ([(p*4 + t)*C + c][n][H][W]), so each of the
// 4*C loads is coalesced across the warp (consecutive X).
__global__ void __launch_bounds__(128) subpix_gather_kernel(const SubpixGatherArgs a) {
    pdl_wait();
    const int X = static_cast<int>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int row = static_cast<int>(blockIdx.y);
    const int p = static_cast<int>(blockIdx.z);
    const int n = row / a.H, Y = row - n * a.H;
    if (X >= a.W) return;
    const int py = p >> 1, px = p & 1;
    const size_t plane = static_cast<size_t>(a.n) * a.H * a.W;  // one y channel
    float acc[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[c] = c < a.C ? __ldg(a.bias + c) : 0.f;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const int sy = Y + (t >> 1) - 1 + py, sx = X + (t & 1) - 1 + px;
        const bool in = sy >= 0 && sy < a.H && sx >= 0 && sx < a.W;
        const float* yp = a.y + (static_cast<size_t>(n) * a.H + (in ? sy : Y)) * a.W + (in ? sx : X) +
                          (p * 4 + t) * a.C * plane;
#pragma unroll
        for (int c = 0; c < 4; ++c)
            if (c < a.C) {
                const float v = __ldg(yp + c * plane);
                acc[c] += in ? v : 0.f;
            }
    }
    const int W2 = 2 * a.W;
    const size_t vplane = static_cast<size_t>(4) * a.H * a.W;  // one video channel
    for (int c = 0; c < a.C; ++c)
        a.out[(static_cast<size_t>(n) * a.C + c) * vplane + static_cast<size_t>(2 * Y + py) * W2 + 2 * X + px] = acc[c];
}

// ------------------------------------------- upsample + thin-output conv
// Last decoder conv fused with its nearest upsample (codec.cpp:103-113):
// one thread per LOW-RES pixel produces the 2x2 output pixels it covers.
// Per output parity (py,px) the 3x3 conv over the upsampled image is a 2x2
// conv over the low-res image with merged taps (sub-pixel decomposition);
// the 3x3 low-res neighbourhood feeds 16 (parity, tap) pairs.  Merged
// weights wm[p][dy*2+dx][c][4] (COUT <= 4, zero padded) are prepared on the
// host and read as one 16-byte shared-memory vector per (pair, channel).
// Each thread covers two horizontally adjacent low-res pixels so every
// weight vector feeds 2 pixels x COUT FMAs.
template <int COUT>
__global__ void __launch_bounds__(128) upconv_thin_kernel(const UpThinArgs a) {
    extern __shared__ float4 wsm4[];
    const int nw = 16 * a.c_in;
    for (int i = threadIdx.x; i < nw; i += blockDim.x) wsm4[i] = reinterpret_cast<const float4*>(a.wm)[i];
    __syncthreads();
    const int H = 2 * a.Hin, W = 2 * a.Win;
    const int wpairs = (a.Win + 1) / 2;
    const int64_t total = static_cast<int64_t>(a.nimg) * a.Hin * wpairs;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int X0 = 2 * static_cast<int>(idx % wpairs);
        const int Y = static_cast<int>((idx / wpairs) % a.Hin);
        const int n = static_cast<int>(idx / (static_cast<int64_t>(wpairs) * a.Hin));
        float acc[2][4][COUT];
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
            for (int p = 0; p < 4; ++p)
#pragma unroll
                for (int o = 0; o < COUT; ++o) acc[q][p][o] = 0.0f;
        const __half* base = a.x + static_cast<int64_t>(n) * a.Hin * a.Win * a.cs_in;
        for (int c0 = 0; c0 < a.c_in; c0 += 8) {
            // 3 rows x 4 columns (X0-1 .. X0+2) of 8-channel vectors
            uint4 nb[3][4];
#pragma unroll
            for (int ry = 0; ry < 3; ++ry) {
                const int iy = Y + ry - 1;
#pragma unroll
                for (int cx = 0; cx < 4; ++cx) {
                    const int ix = X0 + cx - 1;
                    if (iy >= 0 && iy < a.Hin && ix >= 0 && ix < a.Win)
                        nb[ry][cx] = *reinterpret_cast<const uint4*>(
                            base + (static_cast<int64_t>(iy) * a.Win + ix) * a.cs_in + c0);
                    else
                        nb[ry][cx] = make_uint4(0, 0, 0, 0);
                }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (c0 + j >= a.c_in) break;
                float v[3][4];
#pragma unroll
                for (int ry = 0; ry < 3; ++ry)
#pragma unroll
                    for (int cx = 0; cx < 4; ++cx)
                        v[ry][cx] = __half2float(reinterpret_cast<const __half*>(&nb[ry][cx])[j]);
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                    const int py = p / 2, px = p % 2;
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const int dy = t / 2, dx = t % 2;
                        const float4 w = wsm4[(p * 4 + t) * a.c_in + c0 + j];
                        const int ry = dy - 1 + py + 1;  // row index into nb
#pragma unroll
                        for (int q = 0; q < 2; ++q) {
                            const float x = v[ry][q + dx - 1 + px + 1];
                            acc[q][p][0] = fmaf(w.x, x, acc[q][p][0]);
                            if (COUT > 1) acc[q][p][1 % COUT] = fmaf(w.y, x, acc[q][p][1 % COUT]);
                            if (COUT > 2) acc[q][p][2 % COUT] = fmaf(w.z, x, acc[q][p][2 % COUT]);
                            if (COUT > 3) acc[q][p][3 % COUT] = fmaf(w.w, x, acc[q][p][3 % COUT]);
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            if (X0 + q >= a.Win) break;
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                const int oy = 2 * Y + p / 2, ox = 2 * (X0 + q) + p % 2;
#pragma unroll
                for (int o = 0; o < COUT; ++o)
                    a.out[((static_cast<int64_t>(n) * COUT + o) * H + oy) * W + ox] = acc[q][p][o] + a.bias[o];
            }
        }
    }
}

// ------------------------------------------------------------ thin output
// One thread per output pixel, all (<= 8) output channels; taps outer,
// channels inner with 16-byte fp16 loads.  Weights in shared memory as
// [ky][kx][ic][c_out].
template <int COUT>
__global__ void thin_out_kernel(const ThinOutArgs a) {
    extern __shared__ float wsm[];
    const int kk = a.k * a.k;
    const int nw = COUT * a.c_in * kk;
    for (int i = threadIdx.x; i < nw; i += blockDim.x) {
        const int oc = i / (a.c_in * kk), rest = i % (a.c_in * kk);
        const int ic = rest / kk, t = rest % kk;
        wsm[(t * a.c_in + ic) * COUT + oc] = a.w[i];
    }
    __syncthreads();
    const int H = a.up2 ? 2 * a.Hin : a.Hin, W = a.up2 ? 2 * a.Win : a.Win;
    const int oh = a.win.oy1 - a.win.oy0, ow = a.win.ox1 - a.win.ox0;
    const int64_t total = static_cast<int64_t>(a.nimg) * oh * ow;
    const int r = (a.k - 1) / 2;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int ox = a.win.ox0 + static_cast<int>(idx % ow);
        const int oy = a.win.oy0 + static_cast<int>((idx / ow) % oh);
        const int n = static_cast<int>(idx / (static_cast<int64_t>(ow) * oh));
        float acc[COUT];
#pragma unroll
        for (int o = 0; o < COUT; ++o) acc[o] = 0.0f;
        for (int ky = 0; ky < a.k; ++ky) {
            const int uy = oy + ky - r;
            if (uy < a.win.vy0 || uy >= a.win.vy1) continue;
            const int iy = a.up2 ? (uy >> 1) : uy;
            for (int kx = 0; kx < a.k; ++kx) {
                const int ux = ox + kx - r;
                if (ux < a.win.vx0 || ux >= a.win.vx1) continue;
                const int ix = a.up2 ? (ux >> 1) : ux;
                const __half* px = a.x + ((static_cast<int64_t>(n) * a.Hin + iy) * a.Win + ix) * a.cs_in;
                const float* wt = wsm + (ky * a.k + kx) * a.c_in * COUT;
                for (int c0 = 0; c0 < a.c_in; c0 += 8) {
                    const uint4 raw = *reinterpret_cast<const uint4*>(px + c0);
                    const __half2* h2 = reinterpret_cast<const __half2*>(&raw);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        float2 f = __half22float2(h2[j]);
                        if (a.apply_affine) {
                            f.x = f.x * a.s + a.o;
                            f.y = f.y * a.s + a.o;
                        }
                        const int c = c0 + 2 * j;
                        if (c < a.c_in) {
#pragma unroll
                            for (int o = 0; o < COUT; ++o) acc[o] = fmaf(wt[c * COUT + o], f.x, acc[o]);
                        }
                        if (c + 1 < a.c_in) {
#pragma unroll
                            for (int o = 0; o < COUT; ++o) acc[o] = fmaf(wt[(c + 1) * COUT + o], f.y, acc[o]);
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int o = 0; o < COUT; ++o)
            a.out[((static_cast<int64_t>(n) * COUT + o) * H + oy) * W + ox] = acc[o] + a.bias[o];
    }
}

// ------------------------------------------------------------- resampling
__global__ void down2_kernel(const __half* __restrict__ in, __half* __restrict__ out, int nimg,
                             int H, int W, int cs) {
    pdl_wait();
    const int h2 = H / 2, w2 = W / 2, cv = cs / 8;
    const int64_t total = static_cast<int64_t>(nimg) * h2 * w2 * cv;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int c8 = static_cast<int>(i % cv);
        int64_t p = i / cv;
        const int x = static_cast<int>(p % w2);
        p /= w2;
        const int y = static_cast<int>(p % h2);
        const int n = static_cast<int>(p / h2);
        const __half* r0 = in + ((static_cast<int64_t>(n) * H + 2 * y) * W + 2 * x) * cs + c8 * 8;
        const __half* r1 = r0 + static_cast<int64_t>(W) * cs;
        const uint4 a = *reinterpret_cast<const uint4*>(r0);
        const uint4 b = *reinterpret_cast<const uint4*>(r0 + cs);
        const uint4 c = *reinterpret_cast<const uint4*>(r1);
        const uint4 d = *reinterpret_cast<const uint4*>(r1 + cs);
        const __half2* ha = reinterpret_cast<const __half2*>(&a);
        const __half2* hb = reinterpret_cast<const __half2*>(&b);
        const __half2* hc = reinterpret_cast<const __half2*>(&c);
        const __half2* hd = reinterpret_cast<const __half2*>(&d);
        __align__(16) __half2 o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float2 fa = __half22float2(ha[j]), fb = __half22float2(hb[j]);
            const float2 fc = __half22float2(hc[j]), fd = __half22float2(hd[j]);
            o[j] = __floats2half2_rn(0.25f * (((fa.x + fb.x) + fc.x) + fd.x),
                                     0.25f * (((fa.y + fb.y) + fc.y) + fd.y));
        }
        *reinterpret_cast<uint4*>(out + ((static_cast<int64_t>(n) * h2 + y) * w2 + x) * cs + c8 * 8) =
            *reinterpret_cast<uint4*>(o);
    }
}

__global__ void up2_kernel(const __half* __restrict__ in, __half* __restrict__ out, int nimg, int H,
                           int W, int cs) {
    const int H2 = 2 * H, W2 = 2 * W, cv = cs / 8;
    const int64_t total = static_cast<int64_t>(nimg) * H2 * W2 * cv;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int c8 = static_cast<int>(i % cv);
        int64_t p = i / cv;
        const int x = static_cast<int>(p % W2);
        p /= W2;
        const int y = static_cast<int>(p % H2);
        const int n = static_cast<int>(p / H2);
        *reinterpret_cast<uint4*>(out + ((static_cast<int64_t>(n) * H2 + y) * W2 + x) * cs + c8 * 8) =
            *reinterpret_cast<const uint4*>(in + ((static_cast<int64_t>(n) * H + y / 2) * W + x / 2) * cs +
                                            c8 * 8);
    }
}

// ------------------------------------------------------------ step update
__global__ void step_kernel(const StepArgs a) {
    pdl_wait();
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < a.n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const float eu = a.eps2[i], ec = a.eps2[a.n + i];
        const float eps = __fadd_rn(__fmul_rn(1.0f - a.g, eu), __fmul_rn(a.g, ec));
        float xn = __fadd_rn(__fmul_rn(a.a, a.x[i]), __fmul_rn(a.b, eps));
        if (a.z) xn = __fadd_rn(__fmul_rn(1.0f, xn), __fmul_rn(a.c, a.z[i]));
        a.x_out[i] = xn;
        if (!isfinite(xn)) atomicOr(a.bad, 1);
    }
}

__global__ void linear_kernel(float a, const float* x, float b, const float* y, float* out, int64_t n) {
    pdl_wait();
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = __fadd_rn(__fmul_rn(a, x[i]), __fmul_rn(b, y[i]));
}

__global__ void isfinite_kernel(const float* x, int64_t n, int* bad) {
    pdl_wait();
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        if (!isfinite(x[i])) atomicOr(bad, 1);
}

int grid_for(int64_t work, int threads) {
    const int64_t blocks = (work + threads - 1) / threads;
    return static_cast<int>(blocks < 148 * 32 ? (blocks < 1 ? 1 : blocks) : 148 * 32);
}

}  // namespace

template <int MAXIN>
static cudaError_t launch_thin_in_fast(const ThinInArgs& a, cudaStream_t st) {
    const int cpad8 = (a.c_out + 7) / 8 * 8;
    const size_t smem = sizeof(float) * static_cast<size_t>((a.c_in * a.k * a.k + 1) * cpad8);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(thin_in_fast_kernel<MAXIN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    const int nimg = a.cfg_pair ? 2 * a.nsrc : a.nsrc;
    const int64_t work = 8 * static_cast<int64_t>(nimg) * (a.win.oy1 - a.win.oy0) * (a.win.ox1 - a.win.ox0);
    thin_in_fast_kernel<MAXIN><<<grid_for(work, 128), 128, smem, st>>>(a, cpad8);
    return cudaGetLastError();
}

cudaError_t launch_patch(const ThinInArgs& a, int kp, cudaStream_t st) {
    const int nimg = a.cfg_pair ? 2 * a.nsrc : a.nsrc;
    const int64_t work =
        static_cast<int64_t>(nimg) * (a.win.oy1 - a.win.oy0) * (a.win.ox1 - a.win.ox0) * (kp / 8);
    const int rows = nimg * (a.win.oy1 - a.win.oy0);
    if (a.k == 3 && kp == 64 && a.c_in * 9 <= 64) {
        const int64_t px = static_cast<int64_t>(rows) * (a.win.ox1 - a.win.ox0);
        if (px <= 0) return cudaSuccess;
        // small launches (a decoder slice): narrower blocks to fill the SMs
        const int tb = px < 4 * 148 * 256 ? 64 : 256;
        const dim3 grid(static_cast<unsigned>((px + tb - 1) / tb)), blk(tb);
        switch (a.c_in) {
            case 1: return launch_pdl(patch3_kernel<1>, grid, blk, 0, st, a);
            case 2: return launch_pdl(patch3_kernel<2>, grid, blk, 0, st, a);
            case 3: return launch_pdl(patch3_kernel<3>, grid, blk, 0, st, a);
            case 4: return launch_pdl(patch3_kernel<4>, grid, blk, 0, st, a);
            case 5: return launch_pdl(patch3_kernel<5>, grid, blk, 0, st, a);
            case 6: return launch_pdl(patch3_kernel<6>, grid, blk, 0, st, a);
            case 7: return launch_pdl(patch3_kernel<7>, grid, blk, 0, st, a);
            default: break;
        }
    }
    return launch_pdl(patch_kernel, dim3(grid_for(work, 256)), dim3(256), 0, st, a, kp);
}

cudaError_t launch_tap_gather(const TapGatherArgs& a, cudaStream_t st) {
    const int ow = a.win.ox1 - a.win.ox0, rows = a.n * (a.win.oy1 - a.win.oy0);
    if (ow <= 0 || rows <= 0) return cudaSuccess;
    if (a.C > 4) return cudaErrorInvalidValue;
    const int64_t total = static_cast<int64_t>(rows) * ow;
    if (total >= (int64_t{1} << 31)) return cudaErrorInvalidValue;
    const dim3 grid(static_cast<unsigned>((total + 255) / 256), a.C);
    switch (a.k) {
        case 1: return launch_pdl(tap_gather_kernel<1>, grid, dim3(256), 0, st, a);
        case 3: return launch_pdl(tap_gather_kernel<3>, grid, dim3(256), 0, st, a);
        case 5: return launch_pdl(tap_gather_kernel<5>, grid, dim3(256), 0, st, a);
        case 7: return launch_pdl(tap_gather_kernel<7>, grid, dim3(256), 0, st, a);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_subpix_gather(const SubpixGatherArgs& a, cudaStream_t st) {
    const int rows = a.n * a.H;
    if (a.W <= 0 || rows <= 0) return cudaSuccess;
    if (a.C > 4 || rows >= 65536) return cudaErrorInvalidValue;
    return launch_pdl(subpix_gather_kernel, dim3((a.W + 127) / 128, rows, 4), dim3(128), 0, st, a);
}

cudaError_t launch_upconv_thin(const UpThinArgs& a, cudaStream_t st) {
    const size_t smem = sizeof(float) * static_cast<size_t>(16 * a.c_in * 4);
    const int64_t work = static_cast<int64_t>(a.nimg) * a.Hin * ((a.Win + 1) / 2);
#define LC_UPTHIN(N)                                                                                \
    case N: {                                                                                       \
        if (smem > 48 * 1024) {                                                                     \
            cudaError_t e = cudaFuncSetAttribute(upconv_thin_kernel<N>,                             \
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                                                 static_cast<int>(smem));                           \
            if (e != cudaSuccess) return e;                                                         \
        }                                                                                           \
        upconv_thin_kernel<N><<<grid_for(work, 128), 128, smem, st>>>(a);                           \
        break;                                                                                      \
    }
    switch (a.c_out) {
        LC_UPTHIN(1)
        LC_UPTHIN(2)
        LC_UPTHIN(3)
        LC_UPTHIN(4)
        default: return cudaErrorInvalidValue;
    }
#undef LC_UPTHIN
    return cudaGetLastError();
}

cudaError_t launch_thin_in(const ThinInArgs& a, cudaStream_t st) {
    const int kk_in = a.c_in * a.k * a.k;
    if (a.cs_out % 8 == 0) {
        if (kk_in <= 9) return launch_thin_in_fast<9>(a, st);
        if (kk_in <= 36) return launch_thin_in_fast<36>(a, st);
        if (kk_in <= 64) return launch_thin_in_fast<64>(a, st);
    }
    const size_t smem = sizeof(float) * static_cast<size_t>(a.c_out * a.c_in * a.k * a.k);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(thin_in_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    const int nimg = a.cfg_pair ? 2 * a.nsrc : a.nsrc;
    const int64_t work = static_cast<int64_t>(nimg) * (a.win.oy1 - a.win.oy0) * (a.win.ox1 - a.win.ox0) * a.c_out;
    thin_in_kernel<<<grid_for(work, 256), 256, smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_thin_out(const ThinOutArgs& a, cudaStream_t st) {
    const size_t smem = sizeof(float) * static_cast<size_t>(8 * a.c_in * a.k * a.k);
    const int64_t work = static_cast<int64_t>(a.nimg) * (a.win.oy1 - a.win.oy0) * (a.win.ox1 - a.win.ox0);
    const int grid = grid_for(work, 128);
#define LC_THIN_OUT(N)                                                                              \
    case N: {                                                                                       \
        if (smem > 48 * 1024) {                                                                     \
            cudaError_t e = cudaFuncSetAttribute(thin_out_kernel<N>,                                \
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                                                 static_cast<int>(smem));                           \
            if (e != cudaSuccess) return e;                                                         \
        }                                                                                           \
        thin_out_kernel<N><<<grid, 128, smem, st>>>(a);                                             \
        break;                                                                                      \
    }
    switch (a.c_out) {
        LC_THIN_OUT(1)
        LC_THIN_OUT(2)
        LC_THIN_OUT(3)
        LC_THIN_OUT(4)
        LC_THIN_OUT(5)
        LC_THIN_OUT(6)
        LC_THIN_OUT(7)
        LC_THIN_OUT(8)
        default: return cudaErrorInvalidValue;
    }
#undef LC_THIN_OUT
    return cudaGetLastError();
}

cudaError_t launch_down2(const __half* in, __half* out, int nimg, int H, int W, int cs, cudaStream_t st) {
    const int64_t work = static_cast<int64_t>(nimg) * (H / 2) * (W / 2) * (cs / 8);
    return launch_pdl(down2_kernel, dim3(grid_for(work, 256)), dim3(256), 0, st, in, out, nimg, H, W, cs);
}

cudaError_t launch_up2(const __half* in, __half* out, int nimg, int H, int W, int cs, cudaStream_t st) {
    const int64_t work = static_cast<int64_t>(nimg) * 4 * H * W * (cs / 8);
    up2_kernel<<<grid_for(work, 256), 256, 0, st>>>(in, out, nimg, H, W, cs);
    return cudaGetLastError();
}

cudaError_t launch_step(const StepArgs& a, cudaStream_t st) {
    return launch_pdl(step_kernel, dim3(grid_for(a.n, 256)), dim3(256), 0, st, a);
}

cudaError_t launch_linear(float a, const float* x, float b, const float* y, float* out, int64_t n,
                          cudaStream_t st) {
    return launch_pdl(linear_kernel, dim3(grid_for(n, 256)), dim3(256), 0, st, a, x, b, y, out, n);
}

cudaError_t launch_isfinite(const float* x, int64_t n, int* bad, cudaStream_t st) {
    return launch_pdl(isfinite_kernel, dim3(grid_for(n, 256)), dim3(256), 0, st, x, n, bad);
}

}  // namespace lc
