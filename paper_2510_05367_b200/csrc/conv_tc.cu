// tcgen05 implicit-GEMM convolution kernel.  See conv_tc.cuh for the design.
//
// Persistent, warp-specialised: one CTA (or CTA pair) per SM walks the tile
// list (M tiles fastest so co-resident CTAs share the weight tile in L2).
//   warp 0      TMA producer: A (activation box per tap) + B (weights) into a
//               smem ring (mbarrier full/empty pairs);
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer, fp32
//               accumulators in TMEM, two accumulator buffers so the
//               epilogue of tile i overlaps the main loop of tile i+1;
//   warps 2..9  epilogue (two warps per TMEM lane quarter, alternating
//               16-column chunks): tcgen05.ld -> scale/shift/bias/SiLU ->
//               fp16 NHWC (or fp32 NCHW) stores, then release the accumulator.
//
// CG = 2 (cta_group::2): a cluster of two CTAs on one TPC computes an M=256
// tile; each CTA stages its own 128 pixel rows of A and HALF of the N rows of
// B, the leader CTA issues the 256xN MMAs, each CTA's TMEM receives its own
// 128 rows of the accumulator.  Per SM this halves the B staging traffic and
// the shared-memory bytes read per MMA (the single-CTA kernel is close to
// smem-bandwidth bound at BN <= 160).
#include "conv_tc.cuh"
#include "ptx.cuh"

namespace lc {

namespace {

constexpr int kBM = 128;           // UMMA M per CTA (pixels per tile, padded)
constexpr int kBK = 64;            // K elements per stage (one 128 B row per pixel)
constexpr int kThreads = 320;      // w0 TMA, w1 MMA+TMEM, w2..w9 epilogue
constexpr int kEpiWarps = 8;
constexpr uint32_t kABytes = kBM * kBK * 2;  // 16 KB
constexpr size_t kSmemBudget = 200 * 1024;   // stage ring budget
constexpr int kOffFloats = 5120;             // interior-class offset table (20 KB)

template <int CG>
__host__ __device__ inline int num_stages(int bn) {
    const int per = static_cast<int>(kABytes) + (bn / CG) * kBK * 2;
    int s = static_cast<int>(kSmemBudget / per);
    return s > 8 ? 8 : (s < 2 ? 2 : s);
}

__host__ __device__ inline uint32_t tmem_cols_for(int bn) {
    // two accumulator buffers of bn fp32 columns, power of two >= 32
    const int need = 2 * bn;
    return need <= 32 ? 32u : need <= 64 ? 64u : need <= 128 ? 128u : need <= 256 ? 256u : 512u;
}

// SiLU x*sigmoid(x) = h*(1+tanh(h)), h = x/2: one MUFU.TANH + 2 FP ops.
// tanh.approx has ~2^-11 relative error, below the fp16 rounding of the
// stored activation.
__device__ __forceinline__ float silu_fast(float x) {
    const float h = 0.5f * x;
    float t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(h));
    return fmaf(h, t, h);
}

struct TileCoord {
    int X0, Y0, I0, parity, n_tile;
    bool live;  // M tile exists (the second tile of a pair may not)
};

// Unit u of the schedule -> this CTA's tile.  A unit is CG consecutive M
// tiles (one per CTA of the pair) x one N tile x one parity class.
template <int CG>
__device__ __forceinline__ TileCoord tile_coord(const ConvParams& p, int u, int m_units, int n_tiles, int m_tiles,
                                                int rank) {
    // Operand-stationary order.  Activation-heavy layers: N tile fastest,
    // then parity, then M -- concurrently running CTAs share one input
    // neighbourhood (all N tiles and all four parity classes read the same
    // pixels), fetched from DRAM once while the small weights stay in L2.
    // Weight-heavy layers (deep up blocks: up to 170 MB of per-parity
    // weights): M fastest, so one weight slab is streamed by all CTAs.
    TileCoord c;
    const int P = p.nparity;
    int mu;
    if (p.m_fastest) {
        mu = u % m_units;
        const int rest = u / m_units;
        c.n_tile = rest % n_tiles;
        c.parity = rest / n_tiles;
    } else {
        c.n_tile = u % n_tiles;
        const int rest = u / n_tiles;
        c.parity = rest % P;
        mu = rest / P;
    }
    int mt = mu * CG + rank;
    c.live = mt < m_tiles;
    if (!c.live) mt = m_tiles - 1;  // keep coordinates sane; results are discarded
    const int tx = mt % p.tiles_x;
    mt /= p.tiles_x;
    const int ty = mt % p.tiles_y;
    const int ti = mt / p.tiles_y;
    c.X0 = p.lx0[c.parity] + tx * p.TW;
    c.Y0 = p.ly0[c.parity] + ty * p.TH;
    c.I0 = ti * p.TI;
    return c;
}

template <int CG>
__global__ void __launch_bounds__(kThreads, 1)
    conv_tc_kernel(const __grid_constant__ ConvParams p, int n_tiles, int parities) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte alignment for SW128 atoms.
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    const int stages = num_stages<CG>(p.BN);
    const int bn_cta = p.BN / CG;  // B rows staged by this CTA
    const uint32_t b_bytes = static_cast<uint32_t>(bn_cta) * kBK * 2;
    uint8_t* smA = smem;
    uint8_t* smB = smem + stages * kABytes;
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smB + stages * b_bytes);
    uint64_t* empty_bar = full_bar + stages;
    uint64_t* tfull = empty_bar + stages;  // [2] accumulator ready
    uint64_t* tempty = tfull + 2;          // [2] accumulator drained (leader counts both CTAs)
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
    // per-channel epilogue offsets of the interior border class, bias + o *
    // (sum of all tap weights), per parity: read from shared memory instead of
    // two dependent global loads per 16-channel chunk
    float* off_tab = reinterpret_cast<float*>(smB + stages * b_bytes + 256);

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
    const bool leader = rank == 0;
    const int m_tiles = p.tiles_x * p.tiles_y * p.tiles_i;
    const int m_units = (m_tiles + CG - 1) / CG;
    const int total_units = m_units * n_tiles * parities;
    const int unit0 = static_cast<int>(blockIdx.x) / CG;
    const int unit_step = static_cast<int>(gridDim.x) / CG;

    int total_kb = 0;
    for (int s = 0; s < p.nseg; ++s) total_kb += p.seg[s].ntaps * p.seg[s].ncb;

    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], kEpiWarps * CG);  // one arrive per epilogue warp of the pair
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
        if (CG == 2) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_holder)),
                         "r"(ncols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_holder)),
                         "r"(ncols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    const int rc_rr = p.rc + 1;
    const int n_cls = rc_rr * rc_rr * rc_rr * rc_rr;
    const int cls_int = (p.rc * rc_rr + p.rc) * (rc_rr * rc_rr) + (p.rc * rc_rr + p.rc);
    const bool use_tab = p.shuffle_c == 0 && p.nparity * p.n_pad <= kOffFloats;
    if (use_tab) {
        for (int i = threadIdx.x; i < p.nparity * p.n_pad; i += kThreads) {
            const int par = i / p.n_pad, n = i % p.n_pad;
            off_tab[i] = fmaf(p.shift, p.corr[(static_cast<size_t>(par) * n_cls + cls_int) * p.n_pad + n], p.bias[n]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (CG == 2) cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    const uint32_t acc_stride = ncols / 2;  // column offset of accumulator buffer 1

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (elect_one()) {
            const uint32_t a_bytes = static_cast<uint32_t>(p.TI * p.TH * p.TW) * kBK * 2;
            const uint32_t tx_bytes = CG * (a_bytes + b_bytes);  // both CTAs complete on the leader
            int stage = 0;
            uint32_t phase = 0;
            for (int u = unit0; u < total_units; u += unit_step) {
                const TileCoord tc = tile_coord<CG>(p, u, m_units, n_tiles, m_tiles, static_cast<int>(rank));
                int s = 0, tap = 0, cb = 0;
                int kcoord = p.seg[0].kbase;
                const int nrow = tc.n_tile * p.BN + static_cast<int>(rank) * bn_cta;
                for (int kb = 0; kb < total_kb; ++kb) {
                    mbar_wait(&empty_bar[stage], phase ^ 1);
                    const ConvSegDev& sg = p.seg[s];
                    const int cx = tc.X0 * sg.mx + sg.ox[tc.parity][tap] - sg.wx0;
                    const int cy = tc.Y0 * sg.my + sg.oy[tc.parity][tap] - sg.wy0;
                    if (CG == 1) {
                        mbar_arrive_expect_tx(&full_bar[stage], tx_bytes);
                        tma_load_4d(smA + stage * kABytes, &p.tmA[s], &full_bar[stage], cb * kBK, cx, cy, tc.I0);
                        tma_load_3d(smB + stage * b_bytes, &p.tmB, &full_bar[stage], kcoord, nrow, tc.parity);
                    } else {
                        if (leader) mbar_arrive_expect_tx(&full_bar[stage], tx_bytes);
                        const uint32_t bar = mapa_shared(smem_u32(&full_bar[stage]), 0);
                        tma_load_4d_cg2(smA + stage * kABytes, &p.tmA[s], bar, cb * kBK, cx, cy, tc.I0);
                        tma_load_3d_cg2(smB + stage * b_bytes, &p.tmB, bar, kcoord, nrow, tc.parity);
                    }
                    kcoord += kBK;
                    if (++cb == sg.ncb) {
                        cb = 0;
                        if (++tap == sg.ntaps) {
                            tap = 0;
                            ++s;
                            if (s < p.nseg) kcoord = p.seg[s].kbase;
                        }
                    }
                    if (++stage == stages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (leader CTA)
        if (leader) {
            const uint32_t idesc = umma_idesc_f16(kBM * CG, static_cast<uint32_t>(p.BN));
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int u = unit0; u < total_units; u += unit_step) {
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
                            if (CG == 1)
                                umma_f16(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0 ? 1u : 0u);
                            else
                                umma_f16_cg2(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0 ? 1u : 0u);
                        }
                        if (CG == 1) {
                            umma_commit(&empty_bar[stage]);
                            if (kb == total_kb - 1) umma_commit(&tfull[acc]);
                        } else {
                            umma_commit_cg2(&empty_bar[stage]);
                            if (kb == total_kb - 1) umma_commit_cg2(&tfull[acc]);
                        }
                    }
                    __syncwarp();
                    if (++stage == stages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
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
        const uint32_t tempty_leader[2] = {CG == 2 ? mapa_shared(smem_u32(&tempty[0]), 0) : 0u,
                                           CG == 2 ? mapa_shared(smem_u32(&tempty[1]), 0) : 0u};
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int u = unit0; u < total_units; u += unit_step) {
            const TileCoord tc = tile_coord<CG>(p, u, m_units, n_tiles, m_tiles, static_cast<int>(rank));
            const int img = tc.I0 + li;
            const int Y = tc.Y0 + ly, X = tc.X0 + lx;
            const bool valid = tc.live && (m < p.TI * tile_px) && img < p.n_img && Y < p.ly1[tc.parity] &&
                               X < p.lx1[tc.parity];
            // conditioning-shift border class (distance to the class window)
            int dt = Y - p.cy0, db = p.cy1 - 1 - Y, dl = X - p.cx0, dr = p.cx1 - 1 - X;
            dt = dt < p.rc ? dt : p.rc;
            db = db < p.rc ? db : p.rc;
            dl = dl < p.rc ? dl : p.rc;
            dr = dr < p.rc ? dr : p.rc;
            const int cls = (dt * rr + db) * (rr * rr) + (dl * rr + dr);
            const bool tab = use_tab && (cls == cls_int || !valid);
            const float* corr =
                p.corr + (static_cast<size_t>(tc.parity) * ncls + (valid ? cls : 0)) * p.n_pad;
            const float* tab_row = off_tab + tc.parity * p.n_pad;
            const int oy = Y * p.sy + p.py[tc.parity];
            const int ox = X * p.sx + p.px[tc.parity];
            __half* dst = p.out + ((static_cast<size_t>(img) * p.out_h + oy) * p.out_w + ox) * p.cs_out;

            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const uint32_t t_row = tmem_base + acc * acc_stride + (static_cast<uint32_t>(q * 32) << 16);
            // this warp owns the 16-column chunks eh, eh+2, eh+4, ...; two
            // TMEM loads in flight per wait
            for (int c00 = 16 * eh; c00 < p.BN; c00 += 64) {
                // per-channel offsets bias + o * (sum of in-bound tap weights),
                // loaded before the TMEM wait so the two latencies overlap
                float offv[32];
                if (tab) {
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        const int nb = tc.n_tile * p.BN + c00 + 32 * hh;
                        if (hh == 1 && c00 + 32 >= p.BN) break;
#pragma unroll
                        for (int j = 0; j < 16; j += 4)
                            *reinterpret_cast<float4*>(&offv[16 * hh + j]) =
                                *reinterpret_cast<const float4*>(tab_row + nb + j);
                    }
                } else if (p.shuffle_c == 0) {
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        const int nb = tc.n_tile * p.BN + c00 + 32 * hh;
                        if (hh == 1 && c00 + 32 >= p.BN) break;
#pragma unroll
                        for (int j = 0; j < 16; j += 4) {
                            const float4 cb = *reinterpret_cast<const float4*>(corr + nb + j);
                            const float4 bb = *reinterpret_cast<const float4*>(p.bias + nb + j);
                            offv[16 * hh + j] = fmaf(p.shift, cb.x, bb.x);
                            offv[16 * hh + j + 1] = fmaf(p.shift, cb.y, bb.y);
                            offv[16 * hh + j + 2] = fmaf(p.shift, cb.z, bb.z);
                            offv[16 * hh + j + 3] = fmaf(p.shift, cb.w, bb.w);
                        }
                    }
                }
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
                                    float a = fmaf(__uint_as_float(v[j]), p.scale, offv[16 * hh + j]);
                                    if (p.silu) a = __fdividef(a, 1.0f + __expf(-a));
                                    o32[static_cast<size_t>(nb + j) * plane] = a;
                                }
                            }
                        }
                    } else if (valid && nb < p.cs_out) {
                        const float* off = offv + 16 * hh;
                        __align__(16) __half2 h[8];
#pragma unroll
                        for (int j = 0; j < 16; j += 2) {
                            float a = fmaf(__uint_as_float(v[j]), p.scale, off[j]);
                            float b = fmaf(__uint_as_float(v[j + 1]), p.scale, off[j + 1]);
                            if (p.silu) {
                                a = silu_fast(a);
                                b = silu_fast(b);
                            }
                            h[j / 2] = __floats2half2_rn(a, b);
                        }
                        uint4* d4 = reinterpret_cast<uint4*>(dst + nb);
                        d4[0] = *reinterpret_cast<uint4*>(&h[0]);
                        d4[1] = *reinterpret_cast<uint4*>(&h[4]);
                    }
                }
            }
            // release the accumulator buffer to the MMA warp (the leader's barrier)
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (CG == 1) mbar_arrive(&tempty[acc]);
                else mbar_arrive_cluster(tempty_leader[acc]);
            }
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (CG == 2) cluster_sync();  // peer MMAs into this CTA's TMEM are done
    if (warp == 1) {
        tc_fence_after();
        if (CG == 2)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(ncols));
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(ncols));
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

template <int CG>
size_t smem_bytes_for(int BN) {
    const int st = num_stages<CG>(BN);
    return 1024 + static_cast<size_t>(st) * (kABytes + static_cast<size_t>(BN / CG) * kBK * 2) + 256 +
           kOffFloats * sizeof(float);
}

int g_cta_group_override = -1;  // LC_CTA_GROUP env: 1 or 2 forces the variant

}  // namespace

size_t conv_tc_smem_bytes(int BN) { return smem_bytes_for<1>(BN); }

int conv_tc_cta_group(int BN, int m_tiles, int n_tiles, int parities, int k_blocks) {
    static bool read_env = false;
    if (!read_env) {
        if (const char* v = std::getenv("LC_CTA_GROUP")) g_cta_group_override = std::atoi(v);
        read_env = true;
    }
    // CTA pairs when BN splits into two 16-aligned halves, the main loop is
    // long enough for the smem saving to matter (measured on B200: a win
    // from K = 45 blocks up, a loss at K <= 18 blocks) and there are enough
    // tiles to keep every pair busy.
    const bool ok = BN % 32 == 0 && m_tiles >= 2;
    int cg = (ok && k_blocks >= 32 && m_tiles * n_tiles * parities >= 2 * sm_count()) ? 2 : 1;
    if (g_cta_group_override == 1) cg = 1;
    if (g_cta_group_override == 2 && ok) cg = 2;
    return cg;
}

cudaError_t launch_conv_tc(const ConvParams& p, int parities, cudaStream_t stream) {
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(conv_tc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(kSmemBudget + 2048 + kOffFloats * sizeof(float)));
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(conv_tc_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(kSmemBudget + 2048 + kOffFloats * sizeof(float)));
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    const int n_tiles = p.n_pad / p.BN;
    const int m_tiles = p.tiles_x * p.tiles_y * p.tiles_i;
    const int cg = p.cg;
    if (cg == 1) {
        const int total = m_tiles * n_tiles * parities;
        const int grid = total < sm_count() ? total : sm_count();
        conv_tc_kernel<1><<<grid, kThreads, smem_bytes_for<1>(p.BN), stream>>>(p, n_tiles, parities);
        return cudaGetLastError();
    }
    const int units = ((m_tiles + 1) / 2) * n_tiles * parities;
    const int pairs = units < sm_count() / 2 ? units : sm_count() / 2;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem_bytes_for<2>(p.BN);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, conv_tc_kernel<2>, p, n_tiles, parities);
}

}  // namespace lc
