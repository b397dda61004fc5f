// HBM-bound and thin-channel kernels; see kernels.cuh.
#include "kernels.cuh"

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

__global__ void isfinite_kernel(const float* x, int64_t n, int* bad) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        if (!isfinite(x[i])) atomicOr(bad, 1);
}

int grid_for(int64_t work, int threads) {
    const int64_t blocks = (work + threads - 1) / threads;
    return static_cast<int>(blocks < 148 * 32 ? (blocks < 1 ? 1 : blocks) : 148 * 32);
}

}  // namespace

cudaError_t launch_thin_in(const ThinInArgs& a, cudaStream_t st) {
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
    down2_kernel<<<grid_for(work, 256), 256, 0, st>>>(in, out, nimg, H, W, cs);
    return cudaGetLastError();
}

cudaError_t launch_up2(const __half* in, __half* out, int nimg, int H, int W, int cs, cudaStream_t st) {
    const int64_t work = static_cast<int64_t>(nimg) * 4 * H * W * (cs / 8);
    up2_kernel<<<grid_for(work, 256), 256, 0, st>>>(in, out, nimg, H, W, cs);
    return cudaGetLastError();
}

cudaError_t launch_step(const StepArgs& a, cudaStream_t st) {
    step_kernel<<<grid_for(a.n, 256), 256, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_isfinite(const float* x, int64_t n, int* bad, cudaStream_t st) {
    isfinite_kernel<<<grid_for(n, 256), 256, 0, st>>>(x, n, bad);
    return cudaGetLastError();
}

}  // namespace lc
