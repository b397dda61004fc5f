// tcgen05 implicit-GEMM convolution kernel.  See conv_tc.cuh for the design.
//
// Persistent, warp-specialised: one CTA per SM walks the tile list
// (M tiles fastest so co-resident CTAs share the weight tile in L2).
//   warp 0      TMA producer: A (activation box per tap) + B (weights) into a
//               4-stage smem ring (mbarrier full/empty pairs);
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer, fp32
//               accumulators in TMEM, two accumulator buffers so the
//               epilogue of tile i overlaps the main loop of tile i+1;
//   warps 2..9  epilogue (two warps per TMEM lane quarter, alternating
//               16-column chunks): tcgen05.ld -> scale/shift/bias/SiLU ->
//               fp16 NHWC (or fp32 NCHW) stores, then release the accumulator.
#include "conv_tc.cuh"
#include "ptx.cuh"

namespace lc {

namespace {

constexpr int kBM = 128;           // UMMA M (pixels per tile, padded)
constexpr int kBK = 64;            // K elements per stage (one 128 B row per pixel)
constexpr int kStages = 4;
constexpr int kThreads = 320;      // w0 TMA, w1 MMA+TMEM, w2..w9 epilogue
constexpr int kEpiWarps = 8;
constexpr uint32_t kABytes = kBM * kBK * 2;  // 16 KB

__host__ __device__ inline uint32_t tmem_cols_for(int bn) {
    // two accumulator buffers of bn fp32 columns, power of two >= 32
    const int need = 2 * bn;
    return need <= 32 ? 32u : need <= 64 ? 64u : need <= 128 ? 128u : need <= 256 ? 256u : 512u;
}

struct TileCoord {
    int X0, Y0, I0, parity, n_tile;
};

__device__ __forceinline__ TileCoord tile_coord(const ConvParams& p, int t, int m_tiles, int n_tiles) {
    TileCoord c;
    int mt = t % m_tiles;
    const int rest = t / m_tiles;
    c.n_tile = rest % n_tiles;
    c.parity = rest / n_tiles;
    const int tx = mt % p.tiles_x;
    mt /= p.tiles_x;
    const int ty = mt % p.tiles_y;
    const int ti = mt / p.tiles_y;
    c.X0 = p.lx0[c.parity] + tx * p.TW;
    c.Y0 = p.ly0[c.parity] + ty * p.TH;
    c.I0 = ti * p.TI;
    return c;
}

__global__ void __launch_bounds__(kThreads, 1)
    conv_tc_kernel(const __grid_constant__ ConvParams p, int n_tiles, int parities) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte alignment for SW128 atoms.
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    const uint32_t b_bytes = static_cast<uint32_t>(p.BN) * kBK * 2;
    uint8_t* smA = smem;
    uint8_t* smB = smem + kStages * kABytes;
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smB + kStages * b_bytes);
    uint64_t* empty_bar = full_bar + kStages;
    uint64_t* tfull = empty_bar + kStages;   // [2] accumulator ready
    uint64_t* tempty = tfull + 2;            // [2] accumulator drained
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const int m_tiles = p.tiles_x * p.tiles_y * p.tiles_i;
    const int total_tiles = m_tiles * n_tiles * parities;

    int total_kb = 0;
    for (int s = 0; s < p.nseg; ++s) total_kb += p.seg[s].ntaps * p.seg[s].ncb;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], kEpiWarps);  // one arrive per epilogue warp
        }
        fence_barrier_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&p.tmA[0]);
        if (p.nseg > 1) tma_prefetch_desc(&p.tmA[1]);
        tma_prefetch_desc(&p.tmB);
    }
    const uint32_t ncols = tmem_cols_for(p.BN);
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_holder)),
                     "r"(ncols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    const uint32_t acc_stride = ncols / 2;  // column offset of accumulator buffer 1

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (elect_one()) {
            const uint32_t tx_bytes =
                static_cast<uint32_t>(p.TI * p.TH * p.TW) * kBK * 2 + b_bytes;
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
                const TileCoord tc = tile_coord(p, t, m_tiles, n_tiles);
                int s = 0, tap = 0, cb = 0;
                int kcoord = p.seg[0].kbase;
                const int nrow = tc.n_tile * p.BN;
                for (int kb = 0; kb < total_kb; ++kb) {
                    mbar_wait(&empty_bar[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&full_bar[stage], tx_bytes);
                    const ConvSegDev& sg = p.seg[s];
                    const int cx = tc.X0 * sg.mx + sg.ox[tc.parity][tap] - sg.wx0;
                    const int cy = tc.Y0 * sg.my + sg.oy[tc.parity][tap] - sg.wy0;
                    tma_load_4d(smA + stage * kABytes, &p.tmA[s], &full_bar[stage], cb * kBK, cx, cy,
                                tc.I0);
                    tma_load_3d(smB + stage * b_bytes, &p.tmB, &full_bar[stage], kcoord, nrow,
                                tc.parity);
                    kcoord += kBK;
                    if (++cb == sg.ncb) {
                        cb = 0;
                        if (++tap == sg.ntaps) {
                            tap = 0;
                            ++s;
                            if (s < p.nseg) kcoord = p.seg[s].kbase;
                        }
                    }
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        const uint32_t idesc = umma_idesc_f16(kBM, static_cast<uint32_t>(p.BN));
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
            mbar_wait(&tempty[acc], acc_phase ^ 1);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + acc * acc_stride;
            for (int kb = 0; kb < total_kb; ++kb) {
                mbar_wait(&full_bar[stage], phase);
                tc_fence_after();
                if (elect_one()) {
                    const uint64_t adesc = umma_desc_sw128(smem_u32(smA + stage * kABytes));
                    const uint64_t bdesc = umma_desc_sw128(smem_u32(smB + stage * b_bytes));
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k) {
                        // +32 bytes per K=16 step inside the 128 B swizzle row
                        umma_f16(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0 ? 1u : 0u);
                    }
                    umma_commit(&empty_bar[stage]);
                    if (kb == total_kb - 1) umma_commit(&tfull[acc]);
                }
                __syncwarp();
                if (++stage == kStages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    } else {
        // ------------------------------------------------ epilogue warps
        const int q = warp & 3;          // TMEM lane quarter this warp may access
        const int eh = (warp - 2) >> 2;  // column half: two warps per lane quarter
        const int m = q * 32 + lane;
        const int tile_px = p.TH * p.TW;
        const int li = m / tile_px;
        const int ly = (m / p.TW) % p.TH;
        const int lx = m % p.TW;
        const int rr = p.rc + 1;
        const int ncls = rr * rr * rr * rr;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
            const TileCoord tc = tile_coord(p, t, m_tiles, n_tiles);
            const int img = tc.I0 + li;
            const int Y = tc.Y0 + ly, X = tc.X0 + lx;
            const bool valid = (m < p.TI * tile_px) && img < p.n_img && Y < p.ly1[tc.parity] &&
                               X < p.lx1[tc.parity];
            // conditioning-shift border class (distance to the class window)
            int dt = Y - p.cy0, db = p.cy1 - 1 - Y, dl = X - p.cx0, dr = p.cx1 - 1 - X;
            dt = dt < p.rc ? dt : p.rc;
            db = db < p.rc ? db : p.rc;
            dl = dl < p.rc ? dl : p.rc;
            dr = dr < p.rc ? dr : p.rc;
            const int cls = (dt * rr + db) * (rr * rr) + (dl * rr + dr);
            const float* corr =
                p.corr + (static_cast<size_t>(tc.parity) * ncls + (valid ? cls : 0)) * p.n_pad;
            const int oy = Y * p.sy + p.py[tc.parity];
            const int ox = X * p.sx + p.px[tc.parity];
            __half* dst = p.out + ((static_cast<size_t>(img) * p.out_h + oy) * p.out_w + ox) * p.cs_out;

            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const uint32_t t_row = tmem_base + acc * acc_stride + (static_cast<uint32_t>(q * 32) << 16);
            // this warp owns the 16-column chunks eh, eh+2, eh+4, ...; two
            // TMEM loads in flight per wait
            for (int c00 = 16 * eh; c00 < p.BN; c00 += 64) {
              uint32_t vv[32];
              tmem_ld16(t_row + c00, *reinterpret_cast<uint32_t(*)[16]>(&vv[0]));
              const bool two = c00 + 32 < p.BN;
              if (two) tmem_ld16(t_row + c00 + 32, *reinterpret_cast<uint32_t(*)[16]>(&vv[16]));
              tmem_ld_wait();
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) {
                if (hh == 1 && !two) break;
                const uint32_t* v = vv + 16 * hh;
                const int c0 = c00 + 32 * hh;
                const int nb = tc.n_tile * p.BN + c0;
                if (p.out32 && p.shuffle_c > 0) {
                    // depth-to-space fp32 NCHW (last decoder conv, sub-pixel form)
                    if (valid) {
                        const size_t plane = static_cast<size_t>(p.out_h) * p.out_w;
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            const int ch = nb + j;
                            if (ch < p.c_out) {
                                const int par = ch / p.shuffle_c, o = ch % p.shuffle_c;
                                const float a = __uint_as_float(v[j]) * p.scale + p.bias[ch];
                                p.out32[(static_cast<size_t>(img) * p.shuffle_c + o) * plane +
                                        static_cast<size_t>(2 * Y + par / 2) * p.out_w + 2 * X + par % 2] = a;
                            }
                        }
                    }
                } else if (p.out32) {
                    // fp32 NCHW output (denoiser head: eps feeds the fp32 sampler)
                    if (valid) {
                        const size_t plane = static_cast<size_t>(p.out_h) * p.out_w;
                        float* o32 = p.out32 + (static_cast<size_t>(img) * p.c_out) * plane +
                                     static_cast<size_t>(oy) * p.out_w + ox;
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            if (nb + j < p.c_out) {
                                float a = __uint_as_float(v[j]) * p.scale + p.shift * corr[nb + j] + p.bias[nb + j];
                                if (p.silu) a = __fdividef(a, 1.0f + __expf(-a));
                                o32[static_cast<size_t>(nb + j) * plane] = a;
                            }
                        }
                    }
                } else if (valid && nb < p.cs_out) {
                    // per-channel offset: bias + o * (sum of in-bound tap weights)
                    float off[16];
#pragma unroll
                    for (int j = 0; j < 16; j += 4) {
                        const float4 cb = *reinterpret_cast<const float4*>(corr + nb + j);
                        const float4 bb = *reinterpret_cast<const float4*>(p.bias + nb + j);
                        off[j] = fmaf(p.shift, cb.x, bb.x);
                        off[j + 1] = fmaf(p.shift, cb.y, bb.y);
                        off[j + 2] = fmaf(p.shift, cb.z, bb.z);
                        off[j + 3] = fmaf(p.shift, cb.w, bb.w);
                    }
                    __align__(16) __half2 h[8];
#pragma unroll
                    for (int j = 0; j < 16; j += 2) {
                        float a = fmaf(__uint_as_float(v[j]), p.scale, off[j]);
                        float b = fmaf(__uint_as_float(v[j + 1]), p.scale, off[j + 1]);
                        if (p.silu) {
                            a = __fdividef(a, 1.0f + __expf(-a));
                            b = __fdividef(b, 1.0f + __expf(-b));
                        }
                        h[j / 2] = __floats2half2_rn(a, b);
                    }
                    uint4* d4 = reinterpret_cast<uint4*>(dst + nb);
                    d4[0] = *reinterpret_cast<uint4*>(&h[0]);
                    d4[1] = *reinterpret_cast<uint4*>(&h[4]);
                }
              }
            }
            // release the accumulator buffer to the MMA warp
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(ncols));
    }
}

int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

}  // namespace

size_t conv_tc_smem_bytes(int BN) {
    return 1024 + kStages * (kABytes + static_cast<size_t>(BN) * kBK * 2) + 256;
}

cudaError_t launch_conv_tc(const ConvParams& p, int parities, cudaStream_t stream) {
    const size_t smem = conv_tc_smem_bytes(p.BN);
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(conv_tc_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(conv_tc_smem_bytes(256)));
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    const int n_tiles = p.n_pad / p.BN;
    const int total = p.tiles_x * p.tiles_y * p.tiles_i * n_tiles * parities;
    const int grid = total < sm_count() ? total : sm_count();
    conv_tc_kernel<<<grid, kThreads, smem, stream>>>(p, n_tiles, parities);
    return cudaGetLastError();
}

}  // namespace lc
