// tcgen05 implicit-GEMM convolution kernel.  See conv_tc.cuh for the design.
#include "conv_tc.cuh"
#include "ptx.cuh"

namespace lc {

namespace {

constexpr int kBM = 128;           // UMMA M (pixels per tile, padded)
constexpr int kBK = 64;            // K elements per stage (one 128 B row per pixel)
constexpr int kStages = 4;
constexpr int kThreads = 192;      // w0 TMA, w1 MMA+TMEM, w2..w5 epilogue
constexpr uint32_t kABytes = kBM * kBK * 2;  // 16 KB

__host__ __device__ inline int tmem_cols_for(int bn) {
    return bn <= 32 ? 32 : bn <= 64 ? 64 : bn <= 128 ? 128 : 256;
}

__global__ void __launch_bounds__(kThreads, 1)
    conv_tc_kernel(const __grid_constant__ ConvParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte alignment for SW128 atoms.
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    const uint32_t b_bytes = static_cast<uint32_t>(p.BN) * kBK * 2;
    uint8_t* smA = smem;
    uint8_t* smB = smem + kStages * kABytes;
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smB + kStages * b_bytes);
    uint64_t* empty_bar = full_bar + kStages;
    uint64_t* tmem_full = empty_bar + kStages;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_full + 1);

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;

    // tile coordinates
    const int parity = blockIdx.z;
    const int n_tile = blockIdx.y;
    int mt = blockIdx.x;
    const int tx = mt % p.tiles_x;
    mt /= p.tiles_x;
    const int ty = mt % p.tiles_y;
    const int ti = mt / p.tiles_y;
    const int X0 = p.lx0[parity] + tx * p.TW;
    const int Y0 = p.ly0[parity] + ty * p.TH;
    const int I0 = ti * p.TI;

    int total_kb = 0;
    for (int s = 0; s < p.nseg; ++s) total_kb += p.seg[s].ntaps * p.seg[s].ncb;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], 1);
        }
        mbar_init(tmem_full, 1);
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

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (elect_one()) {
            const uint32_t tx_bytes =
                static_cast<uint32_t>(p.TI * p.TH * p.TW) * kBK * 2 + b_bytes;
            int stage = 0;
            uint32_t phase = 0;
            int s = 0, tap = 0, cb = 0;
            int kcoord = p.seg[0].kbase;
            const int nrow = n_tile * p.BN;
            for (int kb = 0; kb < total_kb; ++kb) {
                mbar_wait(&empty_bar[stage], phase ^ 1);
                mbar_arrive_expect_tx(&full_bar[stage], tx_bytes);
                const ConvSegDev& sg = p.seg[s];
                const int cx = X0 * sg.mx + sg.ox[parity][tap] - sg.wx0;
                const int cy = Y0 * sg.my + sg.oy[parity][tap] - sg.wy0;
                tma_load_4d(smA + stage * kABytes, &p.tmA[s], &full_bar[stage], cb * kBK, cx, cy,
                            I0);
                tma_load_3d(smB + stage * b_bytes, &p.tmB, &full_bar[stage], kcoord, nrow,
                            parity);
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
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        const uint32_t idesc = umma_idesc_f16(kBM, static_cast<uint32_t>(p.BN));
        int stage = 0;
        uint32_t phase = 0;
        for (int kb = 0; kb < total_kb; ++kb) {
            mbar_wait(&full_bar[stage], phase);
            tc_fence_after();
            if (elect_one()) {
                const uint64_t adesc = umma_desc_sw128(smem_u32(smA + stage * kABytes));
                const uint64_t bdesc = umma_desc_sw128(smem_u32(smB + stage * b_bytes));
#pragma unroll
                for (int k = 0; k < kBK / 16; ++k) {
                    // +32 bytes per K=16 step inside the 128 B swizzle row
                    umma_f16(tmem_base, adesc + 2 * k, bdesc + 2 * k, idesc,
                             (kb | k) != 0 ? 1u : 0u);
                }
                umma_commit(&empty_bar[stage]);
                if (kb == total_kb - 1) umma_commit(tmem_full);
            }
            __syncwarp();
            if (++stage == kStages) {
                stage = 0;
                phase ^= 1;
            }
        }
    } else {
        // ------------------------------------------------ epilogue warps
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        const int m = q * 32 + lane;
        const int tile_px = p.TH * p.TW;
        const int li = m / tile_px;
        const int ly = (m / p.TW) % p.TH;
        const int lx = m % p.TW;
        const int img = I0 + li;
        const int Y = Y0 + ly, X = X0 + lx;
        const bool valid = (m < p.TI * tile_px) && img < p.n_img && Y < p.ly1[parity] && X < p.lx1[parity];
        // conditioning-shift border class (distance to the class window)
        const int rr = p.rc + 1;
        int dt = Y - p.cy0, db = p.cy1 - 1 - Y, dl = X - p.cx0, dr = p.cx1 - 1 - X;
        dt = dt < p.rc ? dt : p.rc;
        db = db < p.rc ? db : p.rc;
        dl = dl < p.rc ? dl : p.rc;
        dr = dr < p.rc ? dr : p.rc;
        const int cls = (dt * rr + db) * (rr * rr) + (dl * rr + dr);
        const int ncls = rr * rr * rr * rr;
        const float* corr = p.corr + (static_cast<size_t>(parity) * ncls + (valid ? cls : 0)) * p.n_pad;
        const int oy = Y * p.sy + p.py[parity];
        const int ox = X * p.sx + p.px[parity];
        __half* dst = p.out + ((static_cast<size_t>(img) * p.out_h + oy) * p.out_w + ox) * p.cs_out;

        mbar_wait(tmem_full, 0);
        tc_fence_after();
        const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
        for (int c0 = 0; c0 < p.BN; c0 += 16) {
            uint32_t v[16];
            tmem_ld16(t_row + c0, v);
            tmem_ld_wait();
            const int nb = n_tile * p.BN + c0;
            if (valid && nb < p.cs_out) {
                __align__(16) __half2 h[8];
#pragma unroll
                for (int j = 0; j < 16; j += 2) {
                    float a = __uint_as_float(v[j]) * p.scale + p.shift * corr[nb + j] + p.bias[nb + j];
                    float b = __uint_as_float(v[j + 1]) * p.scale + p.shift * corr[nb + j + 1] +
                              p.bias[nb + j + 1];
                    if (p.silu) {
                        a = a / (1.0f + __expf(-a));
                        b = b / (1.0f + __expf(-b));
                    }
                    h[j / 2] = __floats2half2_rn(a, b);
                }
                uint4* d4 = reinterpret_cast<uint4*>(dst + nb);
                d4[0] = *reinterpret_cast<uint4*>(&h[0]);
                d4[1] = *reinterpret_cast<uint4*>(&h[4]);
            }
        }
        tc_fence_before();
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(ncols));
    }
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
    dim3 grid(p.tiles_x * p.tiles_y * p.tiles_i, n_tiles, parities);
    conv_tc_kernel<<<grid, kThreads, smem, stream>>>(p);
    return cudaGetLastError();
}

}  // namespace lc
