// HBM-bound and thin-channel kernels; see kernels.cuh.
#include "kernels.cuh"
#include "pdl.cuh"

namespace lc {

namespace {


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
    const int nimg = a.cfg_pair ? 2 * a.nsrc : a.nsrc;
    const int idx = min(static_cast<int>(blockIdx.x) * blockDim.x + threadIdx.x, nimg * oh * ow - 1);
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
    // stage the 128-byte row in shared memory (16-byte groups rotated by the
    // thread index: conflict-free), then write the block's rows as one
    // contiguous span (the block's pixels are consecutive in the patch tensor)
    extern __shared__ uint4 rows_sm[];
#pragma unroll
    for (int g = 0; g < 8; ++g) {
        __align__(16) __half2 h[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) h[j] = __floats2half2_rn(v[8 * g + 2 * j], v[8 * g + 2 * j + 1]);
        rows_sm[threadIdx.x * 8 + ((g + threadIdx.x) & 7)] = *reinterpret_cast<const uint4*>(h);
    }
    __syncthreads();
    const int first = static_cast<int>(blockIdx.x) * blockDim.x;
    const int npx = min(static_cast<int>(blockDim.x), nimg * oh * ow - first);
    if (ow == a.W && oh == a.H) {
        // full-image window: the block's pixels are one contiguous span
        uint4* dst = reinterpret_cast<uint4*>(a.out) + static_cast<size_t>(first) * 8;
        for (int i = threadIdx.x; i < npx * 8; i += blockDim.x) {
            const int px = i >> 3, g = i & 7;
            dst[i] = rows_sm[px * 8 + ((g + px) & 7)];
        }
    } else {
        for (int i = threadIdx.x; i < npx * 8; i += blockDim.x) {
            const int px = i >> 3, g = i & 7;
            const int pidx = first + px;
            const int prow = pidx / ow;
            const int pn = prow / oh;
            const int py = a.win.oy0 + (prow - pn * oh), pxx = a.win.ox0 + (pidx - prow * ow);
            reinterpret_cast<uint4*>(a.out + ((static_cast<size_t>(pn) * a.H + py) * a.W + pxx) * 64)[g] =
                rows_sm[px * 8 + ((g + px) & 7)];
        }
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
// One element of the sampler update in the reference's two-rounding order
// (cfg_combine + reverse_step_*, sampler.cpp:95-133).
__device__ __forceinline__ float step_one(const StepArgs& a, float eu, float ec, float x, float z) {
    const float eps = __fadd_rn(__fmul_rn(1.0f - a.g, eu), __fmul_rn(a.g, ec));
    float xn = __fadd_rn(__fmul_rn(a.a, x), __fmul_rn(a.b, eps));
    if (a.z) xn = __fadd_rn(__fmul_rn(1.0f, xn), __fmul_rn(a.c, z));
    return xn;
}

// 16-byte vectors where every operand is 16-byte aligned (the engine's
// buffers are), scalar tail; non-finite results voted per warp.
__global__ void step_kernel(const StepArgs a) {
    pdl_wait();
    int f = 0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    const bool vec = a.n % 4 == 0 && al16(a.eps2) && al16(a.x) && al16(a.x_out) && (!a.z || al16(a.z));
    const int64_t n4 = vec ? a.n / 4 : 0;
    for (int64_t i = tid; i < n4; i += stride) {
        const float4 eu = reinterpret_cast<const float4*>(a.eps2)[i];
        const float4 ec = reinterpret_cast<const float4*>(a.eps2 + a.n)[i];
        const float4 x = reinterpret_cast<const float4*>(a.x)[i];
        const float4 z = a.z ? reinterpret_cast<const float4*>(a.z)[i] : make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 o = make_float4(step_one(a, eu.x, ec.x, x.x, z.x), step_one(a, eu.y, ec.y, x.y, z.y),
                                     step_one(a, eu.z, ec.z, x.z, z.z), step_one(a, eu.w, ec.w, x.w, z.w));
        reinterpret_cast<float4*>(a.x_out)[i] = o;
        f |= !isfinite(o.x) | !isfinite(o.y) | !isfinite(o.z) | !isfinite(o.w);
    }
    for (int64_t i = 4 * n4 + tid; i < a.n; i += stride) {
        const float xn = step_one(a, a.eps2[i], a.eps2[a.n + i], a.x[i], a.z ? a.z[i] : 0.0f);
        a.x_out[i] = xn;
        f |= !isfinite(xn);
    }
    if (__any_sync(0xffffffffu, f) && (threadIdx.x & 31) == 0) atomicOr(a.bad, 1);
}

__global__ void linear_kernel(float a, const float* x, float b, const float* y, float* out, int64_t n) {
    pdl_wait();
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const bool vec = n % 4 == 0 && ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) |
                                     reinterpret_cast<uintptr_t>(out)) & 15) == 0;
    const int64_t n4 = vec ? n / 4 : 0;
    for (int64_t i = tid; i < n4; i += stride) {
        const float4 u = reinterpret_cast<const float4*>(x)[i], v = reinterpret_cast<const float4*>(y)[i];
        reinterpret_cast<float4*>(out)[i] =
            make_float4(__fadd_rn(__fmul_rn(a, u.x), __fmul_rn(b, v.x)), __fadd_rn(__fmul_rn(a, u.y), __fmul_rn(b, v.y)),
                        __fadd_rn(__fmul_rn(a, u.z), __fmul_rn(b, v.z)), __fadd_rn(__fmul_rn(a, u.w), __fmul_rn(b, v.w)));
    }
    for (int64_t i = 4 * n4 + tid; i < n; i += stride) out[i] = __fadd_rn(__fmul_rn(a, x[i]), __fmul_rn(b, y[i]));
}

// all_finite (tensor.cpp:376): 16-byte loads, a per-thread flag and one
// warp-wide vote, so the flag word sees at most one atomic per warp.
__global__ void isfinite_kernel(const float* x, int64_t n, int* bad) {
    pdl_wait();
    int f = 0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const bool aligned = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    const int64_t n4 = aligned ? n / 4 : 0;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    for (int64_t i = tid; i < n4; i += stride) {
        const float4 v = __ldg(x4 + i);
        f |= !isfinite(v.x) | !isfinite(v.y) | !isfinite(v.z) | !isfinite(v.w);
    }
    for (int64_t i = 4 * n4 + tid; i < n; i += stride) f |= !isfinite(x[i]);
    if (__any_sync(0xffffffffu, f) && (threadIdx.x & 31) == 0) atomicOr(bad, 1);
}

int grid_for(int64_t work, int threads) {
    const int64_t blocks = (work + threads - 1) / threads;
    return static_cast<int>(blocks < 148 * 32 ? (blocks < 1 ? 1 : blocks) : 148 * 32);
}

}  // namespace

cudaError_t launch_patch(const ThinInArgs& a, int kp, cudaStream_t st) {
    const int nimg = a.cfg_pair ? 2 * a.nsrc : a.nsrc;
    const int64_t work =
        static_cast<int64_t>(nimg) * (a.win.oy1 - a.win.oy0) * (a.win.ox1 - a.win.ox0) * (kp / 8);
    const int rows = nimg * (a.win.oy1 - a.win.oy0);
    if (a.k == 3 && kp == 64 && a.c_in * 9 <= 64) {
        const int64_t px = static_cast<int64_t>(rows) * (a.win.ox1 - a.win.ox0);
        if (px <= 0) return cudaSuccess;
        // small launches (a decoder slice): narrower blocks to fill the SMs
        const int tb = px < 148 * 256 ? 64 : 256;
        const dim3 grid(static_cast<unsigned>((px + tb - 1) / tb)), blk(tb);
        switch (a.c_in) {
            case 1: return launch_pdl(patch3_kernel<1>, grid, blk, tb * 128, st, a);
            case 2: return launch_pdl(patch3_kernel<2>, grid, blk, tb * 128, st, a);
            case 3: return launch_pdl(patch3_kernel<3>, grid, blk, tb * 128, st, a);
            case 4: return launch_pdl(patch3_kernel<4>, grid, blk, tb * 128, st, a);
            case 5: return launch_pdl(patch3_kernel<5>, grid, blk, tb * 128, st, a);
            case 6: return launch_pdl(patch3_kernel<6>, grid, blk, tb * 128, st, a);
            case 7: return launch_pdl(patch3_kernel<7>, grid, blk, tb * 128, st, a);
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
    return launch_pdl(step_kernel, dim3(grid_for((a.n + 3) / 4, 256)), dim3(256), 0, st, a);
}

cudaError_t launch_linear(float a, const float* x, float b, const float* y, float* out, int64_t n,
                          cudaStream_t st) {
    return launch_pdl(linear_kernel, dim3(grid_for((n + 3) / 4, 256)), dim3(256), 0, st, a, x, b, y, out, n);
}

cudaError_t launch_isfinite(const float* x, int64_t n, int* bad, cudaStream_t st) {
    return launch_pdl(isfinite_kernel, dim3(grid_for((n + 3) / 4, 256)), dim3(256), 0, st, x, n, bad);
}

}  // namespace lc
