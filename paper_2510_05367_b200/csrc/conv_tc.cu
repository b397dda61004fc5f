// tcgen05 implicit-GEMM convolution kernel.  See conv_tc.cuh for the design.
//
// Persistent, warp-specialised: one CTA (or CTA pair) per SM walks the tile
// list (operand-stationary order, see tile_coord).
//   warp 0      TMA producer: A (activation box per tap) + B (weights) into a
//               smem ring (mbarrier full/empty pairs);
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer, fp32
//               accumulators in TMEM, two accumulator buffers so the
//               epilogue of tile i overlaps the main loop of tile i+1;
//   warps 2..9  epilogue (two warps per TMEM lane quarter, alternating
//               16-column chunks): tcgen05.ld -> scale/offset/SiLU ->
//               fp16 NHWC (or fp32 NCHW) stores, then release the accumulator.
//
// Epilogue offsets.  The folded conditioning needs, per output channel and
// per pixel border class, off = bias + o * (sum of in-bound tap weights).  The
// epilogue warps stage the (parity, N tile) slice of that table for the NEXT
// tile in shared memory with cp.async while they drain the current one, so the
// inner loop reads offsets with broadcast ld.shared instead of two dependent
// global loads per 16-column chunk (the stem GEMM went from 66 to ~46 us on
// that alone).  The SiLU half-argument (x*sigmoid(x) = h + h*tanh(h), h = x/2)
// is folded into the staged offsets and the scale.
//
// CG = 2 (cta_group::2): a cluster of two CTAs on one TPC computes an M=256
// tile; each CTA stages its own 128 pixel rows of A and HALF of the N rows of
// B, the leader CTA issues the 256xN MMAs, each CTA's TMEM receives its own
// 128 rows of the accumulator.  Per SM this halves the B staging traffic and
// the shared-memory bytes read per MMA (the single-CTA kernel is close to
// smem-bandwidth bound at BN <= 160).
#include "conv_tc.cuh"
#include "ptx.cuh"
#include "pdl.cuh"

#include <cstdlib>

namespace lc {

namespace {

constexpr int kBM = 128;           // UMMA M per CTA (pixels per tile, padded)
constexpr int kBK = 64;            // K elements per stage (one 128 B row per pixel)
#ifndef LC_EPI_WARPS
#define LC_EPI_WARPS 16
#endif
constexpr int kEpiWarps = LC_EPI_WARPS;             // epilogue warps: 4 TMEM lane quarters x kEpiGroups
constexpr int kEpiGroups = kEpiWarps / 4;           // warps sharing one lane quarter (column groups)
constexpr int kChunks = kEpiWarps >= 16 ? 1 : 2;    // 16-column chunks per TMEM wait (register budget)
constexpr int kPair = 16 * kEpiGroups;              // column distance of a warp's consecutive chunks
constexpr int kThreads = 64 + kEpiWarps * 32;       // w0 TMA, w1 MMA+TMEM, w2.. epilogue
constexpr int kEpiThreads = kEpiWarps * 32;
constexpr uint32_t kABytes = kBM * kBK * 2;  // 16 KB
constexpr int kSmemMax = 232448;             // 227 KB opt-in dynamic shared memory
constexpr int kSmemFixed = 1024 + 256;       // alignment slack + barriers
constexpr int kMaxTabClasses = 16;           // border classes staged in smem (3x3 kernels)

// Epilogue flavours (compile-time, so the inner loop carries no mode tests).
enum Epi : int {
    kEpiF16 = 0,      // fp16 NHWC
    kEpiF16Silu = 1,  // fp16 NHWC, SiLU
    kEpiF32 = 2,      // fp32 NCHW (denoiser head)
    kEpiShuffle = 3,  // fp32 NCHW depth-to-space (last decoder conv)
    kEpiF32Raw = 4,   // fp32 NHWC, scale * acc only (tap-to-N GEMMs)
};

// floats of one staged offset table: ncls class rows + the bias row, BN wide
__host__ __device__ inline int tab_floats(int rc, int bn) {
    const int rr = rc + 1;
    const int ncls = rr * rr * rr * rr;
    return ncls <= kMaxTabClasses ? (ncls + 1) * bn : 0;
}

// one staged TMA-store box: 32 px x 16 channels (fp32 raw or fp16)
__host__ __device__ inline int stage_chunk(int wide) { return wide ? 2048 : 1024; }
// TMA-store staging slots per epilogue warp: one per chunk of a TMEM wait,
// or (one chunk per wait, fp32 raw output) a 2-slot ring so the next box is
// staged while the previous one is still being read by the TMA unit
__host__ __device__ inline int stage_slots(int wide) { return (kChunks == 2 || wide) ? 2 : 1; }
// offset tables: double-buffered, single with a weight-stationary schedule
// (one (parity, N tile) slab per CTA)
__host__ __device__ inline int tab_bytes(int tabf, int b_res) { return (b_res ? 1 : 2) * tabf * 4; }
__host__ __device__ inline int epi_smem_bytes(int tabf, int tma_out, int wide, int b_res) {
    // offset tables, then (1024-aligned) the TMA-store staging (2 boxes per epilogue warp)
    const int tb = tab_bytes(tabf, b_res);
    return tma_out ? ((tb + 1023) & ~1023) + kEpiWarps * stage_slots(wide) * stage_chunk(wide) : tb;
}

// ring stages: A + B per stage, or A only with a resident weight panel of
// total_kb K blocks (b_res)
// A-operand bytes of one ring stage: one 128-pixel box, or (halo staging)
// one hh x hw box rounded up to the 1024 B swizzle atom
__host__ __device__ inline int a_stage_bytes(const ConvParams& p) {
    return p.halo ? (p.hw * p.hh * kBK * 2 + 1023) & ~1023 : static_cast<int>(kABytes);
}

template <int CG>
__host__ __device__ inline int num_stages(int bn, int tabf, int tma_out, int b_res, int total_kb, int wide,
                                          int a_stage) {
    const int bblk = (bn / CG) * kBK * 2;
    const int per = a_stage + (b_res ? 0 : bblk);
    int s = (kSmemMax - kSmemFixed - epi_smem_bytes(tabf, tma_out, wide, b_res) - (b_res ? total_kb * bblk : 0)) / per;
    return s > 8 ? 8 : (s < 2 ? 2 : s);
}

// Halo staging without a resident weight panel: separate rings, kHaloAStages
// halo boxes (one per channel block, serving every tap) and up to
// 8 - kHaloAStages weight boxes (one per (channel block, tap)); 0 if fewer
// than 3 weight stages fit.
constexpr int kHaloAStages = 2;
template <int CG>
__host__ __device__ inline int halo_ring_bstages(int bn, int tabf, int tma_out, int wide, int a_stage) {
    const int bblk = (bn / CG) * kBK * 2;
    int s = (kSmemMax - kSmemFixed - epi_smem_bytes(tabf, tma_out, wide, 0) - kHaloAStages * a_stage) / bblk;
    s = s > 8 - kHaloAStages ? 8 - kHaloAStages : s;
    return s < 3 ? 0 : s;
}

__host__ __device__ inline uint32_t tmem_cols_for(int bn) {
    // two accumulator buffers of bn fp32 columns, power of two >= 32
    const int need = 2 * bn;
    return need <= 32 ? 32u : need <= 64 ? 64u : need <= 128 ? 128u : need <= 256 ? 256u : 512u;
}

__device__ __forceinline__ float tanh_approx(float x) {
    float t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(x));
    return t;
}

// SiLU x*sigmoid(x) = h*(1+tanh(h)), h = x/2: one MUFU.TANH + 2 FP ops.
// tanh.approx has ~2^-11 relative error, below the fp16 rounding of the
// stored activation.
// SiLU of x = 2h from the half-scaled pre-activation h (the epilogue folds
// the 1/2 into its scale and offsets): 2h * sigmoid(2h) with the exponential
// and reciprocal on the MUFU (ex2.approx / rcp.approx, ~2^-22 relative
// error) instead of tanh.approx (~2^-11): LC_SILU_EXACT=1.
__device__ __forceinline__ float silu_exact_h(float h) {
    const float e = exp2f(-2.8853900817779268f * h);  // exp(-2h), ex2.approx via --use_fast_math-free exp2f
    return __fdividef(2.0f * h, 1.0f + e);
}

__device__ __forceinline__ float silu_fast(float x) {
    const float h = 0.5f * x;
    return fmaf(h, tanh_approx(h), h);
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
    int mu;
    if (p.m_fastest) {
        const int rest = p.fd_units.div(u);
        mu = u - rest * static_cast<int>(p.fd_units.d);
        c.parity = p.fd_ntiles.div(rest);
        c.n_tile = rest - c.parity * static_cast<int>(p.fd_ntiles.d);
    } else {
        const int rest = p.fd_ntiles.div(u);
        c.n_tile = u - rest * static_cast<int>(p.fd_ntiles.d);
        mu = p.fd_par.div(rest);
        c.parity = rest - mu * static_cast<int>(p.fd_par.d);
    }
    (void)m_units;
    (void)n_tiles;
    int mt = mu * CG + rank;
    c.live = mt < m_tiles;
    if (!c.live) mt = m_tiles - 1;  // keep coordinates sane; results are discarded
    const int r1 = p.fd_tx.div(mt);
    const int tx = mt - r1 * static_cast<int>(p.fd_tx.d);
    const int ti = p.fd_ty.div(r1);
    const int ty = r1 - ti * static_cast<int>(p.fd_ty.d);
    c.X0 = p.lx0[c.parity] + tx * p.TW;
    c.Y0 = p.ly0[c.parity] + ty * p.TH;
    c.I0 = ti * p.TI;
    return c;
}

template <int CG, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    conv_tc_kernel(const __grid_constant__ ConvParams p, int n_tiles, int parities) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte alignment for SW128 atoms.
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    int total_kb = 0;
    for (int s = 0; s < p.nseg; ++s) total_kb += p.seg[s].ntaps * p.seg[s].ncb;
    const bool b_res = CG == 1 && p.b_res;
    const int tabf = tab_floats(p.rc, p.BN);
    const bool halo = p.halo;
    const bool halo_ring = halo && !b_res;  // halo boxes + a separate weight ring
    const int a_stage = a_stage_bytes(p);
    const int bstages = halo_ring ? halo_ring_bstages<CG>(p.BN, tabf, p.tma_out, p.nhwc32, a_stage) : 0;
    // ring slots: A+B stages, or kHaloAStages halo stages then bstages weight stages
    const int stages = halo_ring ? kHaloAStages + bstages
                                 : num_stages<CG>(p.BN, tabf, p.tma_out, b_res, total_kb, p.nhwc32, a_stage);
    // fp32 raw (tap-to-N) epilogues need no offset registers: two chunks per wait
    constexpr int kCh = EPI == kEpiF32Raw ? 2 : kChunks;
    const int schunk = stage_chunk(p.nhwc32);
    const int slots = stage_slots(p.nhwc32);
    const bool ring = kCh == 1 && slots == 2;
    const int bn_cta = p.BN / CG;  // B rows staged by this CTA
    const uint32_t b_bytes = static_cast<uint32_t>(bn_cta) * kBK * 2;
    uint8_t* smA = smem;
    uint8_t* smB = smem + (halo_ring ? kHaloAStages : stages) * a_stage;
    const int b_blocks = b_res ? total_kb : (halo_ring ? bstages : stages);  // resident panel or ring
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smB + b_blocks * b_bytes);
    uint64_t* empty_bar = full_bar + stages;
    uint64_t* tfull = empty_bar + stages;  // [2] accumulator ready
    uint64_t* tempty = tfull + 2;          // [2] accumulator drained (leader counts both CTAs)
    uint64_t* bfull = tempty + 2;          // resident weight panel landed (b_res)
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bfull + 1);
    // two epilogue offset tables [ncls + 1][BN] fp32 (see the header comment)
    const uint32_t tab_s = smem_u32(smB + b_blocks * b_bytes + 256);
    // 256 B aligned (tab_s is 1024-aligned + 256): the fp16 staging slots are
    // SWIZZLE_32B TMA-store boxes, whose atom is 256 B
    const uint32_t stage_out_s = tab_s + ((tab_bytes(tabf, b_res) + 1023) & ~1023);

    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x) / 32, 0);  // warp-uniform
    const int lane = threadIdx.x % 32;
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
    const bool leader = rank == 0;
    const int m_tiles = p.tiles_x * p.tiles_y * p.tiles_i;
    const int m_units = (m_tiles + CG - 1) / CG;
    int total_units = m_units * n_tiles * parities;
    int unit0 = static_cast<int>(blockIdx.x) / CG;
    int unit_step = static_cast<int>(gridDim.x) / CG;
    int slab_par = 0, slab_nt = 0;
    if (b_res) {
        // CTA group per (parity, N tile) slab; units are that slab's M tiles
        const int slabs = parities * n_tiles;
        const int cps = static_cast<int>(gridDim.x) / slabs;
        const int slab = static_cast<int>(blockIdx.x) / cps;
        slab_par = slab / n_tiles;
        slab_nt = slab % n_tiles;
        total_units = m_tiles;
        unit0 = static_cast<int>(blockIdx.x) % cps;
        unit_step = cps;
    }
    auto coord = [&](int u) {
        if (!b_res) return tile_coord<CG>(p, u, m_units, n_tiles, m_tiles, static_cast<int>(rank));
        TileCoord c;
        c.parity = slab_par;
        c.n_tile = slab_nt;
        c.live = true;
        const int rest = p.fd_tx.div(u);
        const int tx = u - rest * p.tiles_x;
        const int ti = p.fd_ty.div(rest);
        const int ty = rest - ti * p.tiles_y;
        c.X0 = p.lx0[c.parity] + tx * p.TW;
        c.Y0 = p.ly0[c.parity] + ty * p.TH;
        c.I0 = ti * p.TI;
        return c;
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], kEpiWarps * CG);  // one arrive per epilogue warp of the pair
        }
        mbar_init(bfull, 1);
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
    tc_fence_before();
    __syncthreads();
    if (CG == 2) cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    const uint32_t acc_stride = ncols / 2;  // column offset of accumulator buffer 1
    // everything above overlapped the previous kernel's tail (PDL); inputs
    // and outputs are touched only below
    pdl_trigger();
    pdl_wait();

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (elect_one()) {
            const uint32_t a_bytes = halo ? static_cast<uint32_t>(p.hw * p.hh) * kBK * 2
                                          : static_cast<uint32_t>(p.TI * p.TH * p.TW) * kBK * 2;
            const uint32_t tx_bytes = b_res ? a_bytes : CG * (a_bytes + b_bytes);  // both CTAs complete on the leader
            if (b_res && unit0 < total_units) {
                // the slab's whole weight panel, once (slot = K block of the weight row)
                mbar_arrive_expect_tx(bfull, static_cast<uint32_t>(total_kb) * b_bytes);
                int s = 0, tap = 0, cb = 0, kcoord = p.seg[0].kbase;
                for (int kb = 0; kb < total_kb; ++kb) {
                    tma_load_3d(smB + kb * b_bytes, &p.tmB, bfull, kcoord, slab_nt * p.BN, slab_par);
                    kcoord += kBK;
                    if (++cb == p.seg[s].ncb) {
                        cb = 0;
                        if (++tap == p.seg[s].ntaps) {
                            tap = 0;
                            ++s;
                            if (s < p.nseg) kcoord = p.seg[s].kbase;
                        }
                    }
                }
            }
            int stage = 0;
            uint32_t phase = 0;
            auto advance = [&]() {
                if (++stage == stages) {
                    stage = 0;
                    phase ^= 1;
                }
            };
            if (halo_ring) {
                // halo box per channel block into slots [0, kHaloAStages), then that
                // block's per-tap weight boxes into slots [kHaloAStages, stages)
                const ConvSegDev& sg = p.seg[0];
                int as = 0, bs = 0;
                uint32_t aph = 0, bph = 0;
                for (int u = unit0; u < total_units; u += unit_step) {
                    const TileCoord tc = coord(u);
                    const int nrow = tc.n_tile * p.BN + static_cast<int>(rank) * bn_cta;
                    const int cx = tc.X0 + p.hox[tc.parity] - sg.wx0;
                    const int cy = tc.Y0 + p.hoy[tc.parity] - sg.wy0;
                    for (int cb = 0; cb < sg.ncb; ++cb) {
                        mbar_wait(&empty_bar[as], aph ^ 1);
                        if (CG == 1) {
                            mbar_arrive_expect_tx(&full_bar[as], a_bytes);
                            tma_load_4d(smA + as * a_stage, &p.tmA[0], &full_bar[as], cb * kBK, cx, cy, tc.I0);
                        } else {
                            if (leader) mbar_arrive_expect_tx(&full_bar[as], CG * a_bytes);
                            tma_load_4d_cg2(smA + as * a_stage, &p.tmA[0], mapa_shared(smem_u32(&full_bar[as]), 0),
                                            cb * kBK, cx, cy, tc.I0);
                        }
                        if (++as == kHaloAStages) {
                            as = 0;
                            aph ^= 1;
                        }
                        for (int tap = 0; tap < sg.ntaps; ++tap) {
                            const int slot = kHaloAStages + bs;
                            mbar_wait(&empty_bar[slot], bph ^ 1);
                            const int kcoord = sg.kbase + (tap * sg.ncb + cb) * kBK;
                            if (CG == 1) {
                                mbar_arrive_expect_tx(&full_bar[slot], b_bytes);
                                tma_load_3d(smB + bs * b_bytes, &p.tmB, &full_bar[slot], kcoord, nrow, tc.parity);
                            } else {
                                if (leader) mbar_arrive_expect_tx(&full_bar[slot], CG * b_bytes);
                                tma_load_3d_cg2(smB + bs * b_bytes, &p.tmB, mapa_shared(smem_u32(&full_bar[slot]), 0),
                                                kcoord, nrow, tc.parity);
                            }
                            if (++bs == bstages) {
                                bs = 0;
                                bph ^= 1;
                            }
                        }
                    }
                }
            }
            for (int u = unit0; u < total_units && !halo_ring; u += unit_step) {
                const TileCoord tc = coord(u);
                if (halo) {
                    // one box per channel block serves every tap (see ConvParams::halo)
                    const ConvSegDev& sg = p.seg[0];
                    const int cx = tc.X0 + p.hox[tc.parity] - sg.wx0;
                    const int cy = tc.Y0 + p.hoy[tc.parity] - sg.wy0;
                    for (int cb = 0; cb < sg.ncb; ++cb) {
                        mbar_wait(&empty_bar[stage], phase ^ 1);
                        mbar_arrive_expect_tx(&full_bar[stage], a_bytes);
                        tma_load_4d(smA + stage * a_stage, &p.tmA[0], &full_bar[stage], cb * kBK, cx, cy, tc.I0);
                        advance();
                    }
                    continue;
                }
                const int nrow = tc.n_tile * p.BN + static_cast<int>(rank) * bn_cta;
                // K blocks in (segment, channel block, tap) order
                for (int s = 0; s < p.nseg; ++s) {
                    const ConvSegDev& sg = p.seg[s];
                    for (int cb = 0; cb < sg.ncb; ++cb)
                        for (int tap = 0; tap < sg.ntaps; ++tap) {
                            mbar_wait(&empty_bar[stage], phase ^ 1);
                            const int cx = tc.X0 * sg.mx + sg.ox[tc.parity][tap] - sg.wx0;
                            const int cy = tc.Y0 * sg.my + sg.oy[tc.parity][tap] - sg.wy0;
                            const int kcoord = sg.kbase + (tap * sg.ncb + cb) * kBK;
                            if (CG == 1) {
                                mbar_arrive_expect_tx(&full_bar[stage], tx_bytes);
                                tma_load_4d(smA + stage * a_stage, &p.tmA[s], &full_bar[stage], cb * kBK, cx, cy,
                                            tc.I0);
                                if (!b_res)
                                    tma_load_3d(smB + stage * b_bytes, &p.tmB, &full_bar[stage], kcoord, nrow,
                                                tc.parity);
                            } else {
                                if (leader) mbar_arrive_expect_tx(&full_bar[stage], tx_bytes);
                                const uint32_t bar = mapa_shared(smem_u32(&full_bar[stage]), 0);
                                tma_load_4d_cg2(smA + stage * a_stage, &p.tmA[s], bar, cb * kBK, cx, cy, tc.I0);
                                tma_load_3d_cg2(smB + stage * b_bytes, &p.tmB, bar, kcoord, nrow, tc.parity);
                            }
                            advance();
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
            auto advance = [&]() {
                if (++stage == stages) {
                    stage = 0;
                    phase ^= 1;
                }
            };
            // 128 x BN x 64 from one A stage address and one B panel/ring address
            auto mma_kblock = [&](uint32_t d_tmem, uint32_t a_addr, uint32_t b_addr, bool first) {
                const uint64_t adesc = umma_desc_sw128(a_addr);
                const uint64_t bdesc = umma_desc_sw128(b_addr);
#pragma unroll
                for (int k = 0; k < kBK / 16; ++k) {
                    // +32 bytes per K=16 step inside the 128 B swizzle row
                    const uint32_t accum = (!first || k != 0) ? 1u : 0u;
                    if (CG == 1)
                        umma_f16(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, accum);
                    else
                        umma_f16_cg2(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, accum);
                }
            };
            auto commit = [&](uint64_t* bar) {
                if (CG == 1) umma_commit(bar);
                else umma_commit_cg2(bar);
            };
            int ras = 0, rbs = 0;  // halo_ring slots
            uint32_t raph = 0, rbph = 0;
            if (b_res && unit0 < total_units) mbar_wait(bfull, 0);
            for (int u = unit0; u < total_units; u += unit_step) {
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * acc_stride;
                if (halo_ring) {
                    const ConvSegDev& sg = p.seg[0];
                    const int par = coord(u).parity;
                    for (int cb = 0; cb < sg.ncb; ++cb) {
                        mbar_wait(&full_bar[ras], raph);
                        tc_fence_after();
                        const uint32_t a0 = smem_u32(smA + ras * a_stage);
                        for (int tap = 0; tap < sg.ntaps; ++tap) {
                            const int slot = kHaloAStages + rbs;
                            mbar_wait(&full_bar[slot], rbph);
                            tc_fence_after();
                            if (elect_one()) {
                                const int row = (sg.oy[par][tap] - p.hoy[par]) * p.hw + (sg.ox[par][tap] - p.hox[par]);
                                mma_kblock(d_tmem, a0 + static_cast<uint32_t>(row) * 128u, smem_u32(smB + rbs * b_bytes),
                                           (cb | tap) == 0);
                                commit(&empty_bar[slot]);
                                if (tap == sg.ntaps - 1) {
                                    commit(&empty_bar[ras]);
                                    if (cb == sg.ncb - 1) commit(&tfull[acc]);
                                }
                            }
                            __syncwarp();
                            if (++rbs == bstages) {
                                rbs = 0;
                                rbph ^= 1;
                            }
                        }
                        if (++ras == kHaloAStages) {
                            ras = 0;
                            raph ^= 1;
                        }
                    }
                } else if (halo) {
                    // b_res: every unit of this CTA is its slab's parity
                    const ConvSegDev& sg = p.seg[0];
                    const int par = slab_par;
                    for (int cb = 0; cb < sg.ncb; ++cb) {
                        mbar_wait(&full_bar[stage], phase);
                        tc_fence_after();
                        if (elect_one()) {
                            const uint32_t a0 = smem_u32(smA + stage * a_stage);
                            for (int tap = 0; tap < sg.ntaps; ++tap) {
                                const int row = (sg.oy[par][tap] - p.hoy[par]) * p.hw + (sg.ox[par][tap] - p.hox[par]);
                                mma_kblock(d_tmem, a0 + static_cast<uint32_t>(row) * 128u,
                                           smem_u32(smB + (tap * sg.ncb + cb) * b_bytes), (cb | tap) == 0);
                            }
                            commit(&empty_bar[stage]);
                            if (cb == sg.ncb - 1) commit(&tfull[acc]);
                        }
                        __syncwarp();
                        advance();
                    }
                } else {
                    int kb = 0, seg_kb0 = 0;
                    for (int s = 0; s < p.nseg; ++s) {
                        const ConvSegDev& sg = p.seg[s];
                        for (int cb = 0; cb < sg.ncb; ++cb)
                            for (int tap = 0; tap < sg.ntaps; ++tap, ++kb) {
                                mbar_wait(&full_bar[stage], phase);
                                tc_fence_after();
                                if (elect_one()) {
                                    const int bslot = b_res ? seg_kb0 + tap * sg.ncb + cb : stage;
                                    mma_kblock(d_tmem, smem_u32(smA + stage * a_stage), smem_u32(smB + bslot * b_bytes),
                                               kb == 0);
                                    commit(&empty_bar[stage]);
                                    if (kb == total_kb - 1) commit(&tfull[acc]);
                                }
                                __syncwarp();
                                advance();
                            }
                        seg_kb0 += sg.ntaps * sg.ncb;
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
        const int et = threadIdx.x - 64;  // 0..255
        const int q = warp & 3;           // TMEM lane quarter this warp may access
        const int eg = (warp - 2) >> 2;   // column group: kEpiGroups warps per lane quarter
        const int m = q * 32 + lane;
        const int tile_px = p.TH * p.TW;
        const int li = m / tile_px;
        const int ly = (m / p.TW) % p.TH;
        const int lx = m % p.TW;
        // this warp's first pixel within a tile (TMA-store box origin)
        const int m0_x = (q * 32) % p.TW, m0_y = ((q * 32) / p.TW) % p.TH, m0_i = (q * 32) / tile_px;
        const bool m0_in_tile = q * 32 < p.TI * tile_px;
        const int rr = p.rc + 1;
        const int ncls = rr * rr * rr * rr;
        // SiLU runs on h = x/2: fold the 1/2 into scale and offsets
        constexpr float hs = EPI == kEpiF16Silu ? 0.5f : 1.0f;
        const float hscale = p.scale * hs;
        const uint32_t tempty_leader0 = CG == 2 ? mapa_shared(smem_u32(&tempty[0]), 0) : 0u;
        const uint32_t tempty_leader1 = CG == 2 ? mapa_shared(smem_u32(&tempty[1]), 0) : 0u;
        const int q4 = p.BN / 4;
        // stage the raw corr rows + bias row of (parity, n_tile) into table buf
        auto issue_tab = [&](int buf, int parity, int n_tile) {
            const uint32_t base = tab_s + static_cast<uint32_t>(buf * tabf) * 4u;
            const int nq = (ncls + 1) * q4;
            for (int e = et; e < nq; e += kEpiThreads) {
                const int row = e / q4, c4 = e - row * q4;
                const float* src = row < ncls ? p.corr + (static_cast<size_t>(parity) * ncls + row) * p.n_pad
                                              : p.bias;
                cp_async16(base + static_cast<uint32_t>(e) * 16u, src + n_tile * p.BN + 4 * c4);
            }
            cp_async_commit();
        };
        int cur = 0, cur_key = -1;
        bool pending = false;
        if (tabf && unit0 < total_units) {
            const TileCoord t0 = coord(unit0);
            issue_tab(0, t0.parity, t0.n_tile);
            cur_key = t0.parity * n_tiles + t0.n_tile;
            pending = true;
        }
        int acc = 0;
        uint32_t acc_phase = 0;
        uint32_t stage_it = 0;  // TMA-store staging ring position
        int rot = 0;            // column-group rotation of this tile (ConvParams::epi_rot)
        for (int u = unit0; u < total_units; u += unit_step) {
            const TileCoord tc = coord(u);
            const int egr = kCh == 1 ? (eg + rot) % kEpiGroups : eg;
            rot = (rot + p.epi_rot) % kEpiGroups;
            bool next_switch = false;
            int next_key = cur_key;
            if (tabf) {
                if (pending) {
                    // this tile's slice landed (issued one tile ago): make it
                    // visible, then turn it into hs * (bias + o * corr)
                    cp_async_wait_all();
                    named_bar_sync(1, kEpiThreads);
                    const uint32_t base = tab_s + static_cast<uint32_t>(cur * tabf) * 4u;
                    for (int e = et; e < ncls * q4; e += kEpiThreads) {
                        const int c4 = e % q4;
                        const float4 c = lds128(base + static_cast<uint32_t>(e) * 16u);
                        const float4 b = lds128(base + static_cast<uint32_t>(ncls * q4 + c4) * 16u);
                        sts128(base + static_cast<uint32_t>(e) * 16u,
                               make_float4(hs * fmaf(p.shift, c.x, b.x), hs * fmaf(p.shift, c.y, b.y),
                                           hs * fmaf(p.shift, c.z, b.z), hs * fmaf(p.shift, c.w, b.w)));
                    }
                    named_bar_sync(1, kEpiThreads);
                    pending = false;
                }
                const int un = u + unit_step;
                if (!b_res && un < total_units) {  // one slab per CTA under b_res: never switches
                    const TileCoord tn = coord(un);
                    next_key = tn.parity * n_tiles + tn.n_tile;
                    if (next_key != cur_key) {
                        issue_tab(cur ^ 1, tn.parity, tn.n_tile);
                        next_switch = true;
                    }
                }
            }
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
            const int cls = valid ? (dt * rr + db) * (rr * rr) + (dl * rr + dr) : 0;
            const uint32_t off_row = tab_s + static_cast<uint32_t>(cur * tabf + cls * p.BN) * 4u;
            const float* corr = p.corr + (static_cast<size_t>(tc.parity) * ncls + cls) * p.n_pad;
            const int oy = Y * p.sy + p.py[tc.parity];
            const int ox = X * p.sx + p.px[tc.parity];

            // TMA-store box origin of this warp's 32 pixels (lattice coords
            // relative to the class window, see ConvParams::tmO)
            constexpr bool kF16 = EPI == kEpiF16 || EPI == kEpiF16Silu;
            constexpr bool kTma = kF16 || EPI == kEpiF32Raw;  // epilogues with a TMA-store form
            const bool warp_store = kTma && p.tma_out && tc.live && m0_in_tile;
            const int bx = tc.X0 + m0_x - p.lx0[tc.parity];
            const int by = tc.Y0 + m0_y - p.ly0[tc.parity];
            const int bi = tc.I0 + m0_i;

            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const uint32_t t_row = tmem_base + acc * acc_stride + (static_cast<uint32_t>(q * 32) << 16);
            // this warp owns the 16-column chunks egr, egr+G, egr+2G, ... (G =
            // kEpiGroups); two TMEM loads in flight per wait
            for (int c00 = 16 * egr; c00 < p.BN; c00 += kCh * kPair) {
                const bool two = kCh == 2 && c00 + kPair < p.BN;
                uint32_t vv[16 * kCh];
                tmem_ld16(t_row + c00, *reinterpret_cast<uint32_t(*)[16]>(&vv[0]));
                if (two) tmem_ld16(t_row + c00 + kPair, *reinterpret_cast<uint32_t(*)[16]>(&vv[16 * (kCh - 1)]));
                // offsets hs * (bias + o * corr[class]) for the two chunks
                float offv[16 * kCh];
#pragma unroll
                for (int hh = 0; hh < kCh; ++hh) {
                    if (hh == 1 && !two) break;
                    if (EPI == kEpiF32Raw) break;
                    const int c0 = c00 + kPair * hh;
                    if (tabf) {
#pragma unroll
                        for (int j = 0; j < 16; j += 4)
                            *reinterpret_cast<float4*>(&offv[16 * hh + j]) =
                                lds128(off_row + static_cast<uint32_t>(c0 + j) * 4u);
                    } else {
                        const int nb = tc.n_tile * p.BN + c0;
#pragma unroll
                        for (int j = 0; j < 16; ++j) offv[16 * hh + j] = hs * fmaf(p.shift, corr[nb + j], p.bias[nb + j]);
                    }
                }
                tmem_ld_wait();
                if (kTma && p.tma_out) {
                    // the previous chunk pair's stores have finished reading the staging buffers
                    if (lane == 0) {
                        if (ring) bulk_wait_read1();
                        else bulk_wait_read0();
                    }
                    __syncwarp();
                }
#pragma unroll
                for (int hh = 0; hh < kCh; ++hh) {
                    if (hh == 1 && !two) break;
                    const uint32_t* v = vv + 16 * hh;
                    const float* off = offv + 16 * hh;
                    const int nb = tc.n_tile * p.BN + c00 + kPair * hh;
                    if (EPI == kEpiF32Raw) {
                        if (p.tma_out && p.planar32) {
                            // planar {x, y, img, channel} box: smem [16 ch][32 px], one
                            // conflict-free 4-byte store per channel
                            const uint32_t sb = stage_out_s +
                                                static_cast<uint32_t>(((warp - 2) * slots + (ring ? (stage_it & 1) : hh)) * schunk +
                                                                      lane * 4);
#pragma unroll
                            for (int j = 0; j < 16; ++j)
                                asm volatile("st.shared.f32 [%0], %1;" ::"r"(sb + j * 128u),
                                             "f"(__uint_as_float(v[j]) * hscale)
                                             : "memory");
                        } else if (p.tma_out) {
                            const uint32_t sb =
                                stage_out_s + static_cast<uint32_t>(((warp - 2) * slots + (ring ? (stage_it & 1) : hh)) * schunk + lane * 64);
#pragma unroll
                            for (int j = 0; j < 16; j += 4)
                                sts128(sb + 4 * j, make_float4(__uint_as_float(v[j]) * hscale,
                                                               __uint_as_float(v[j + 1]) * hscale,
                                                               __uint_as_float(v[j + 2]) * hscale,
                                                               __uint_as_float(v[j + 3]) * hscale));
                        } else if (valid && nb < p.cs_out && p.planar32) {
                            const size_t plane = static_cast<size_t>(p.n_img) * p.out_h * p.out_w;
                            const size_t pix = (static_cast<size_t>(img) * p.out_h + oy) * p.out_w + ox;
#pragma unroll
                            for (int j = 0; j < 16; ++j)
                                if (nb + j < p.cs_out) p.out32[(nb + j) * plane + pix] = __uint_as_float(v[j]) * hscale;
                        } else if (valid && nb < p.cs_out) {
                            float4* o4 = reinterpret_cast<float4*>(
                                p.out32 + ((static_cast<size_t>(img) * p.out_h + oy) * p.out_w + ox) * p.cs_out + nb);
#pragma unroll
                            for (int j = 0; j < 16; j += 4)
                                o4[j / 4] = make_float4(__uint_as_float(v[j]) * hscale, __uint_as_float(v[j + 1]) * hscale,
                                                        __uint_as_float(v[j + 2]) * hscale,
                                                        __uint_as_float(v[j + 3]) * hscale);
                        }
                    } else if (EPI == kEpiShuffle) {
                        // depth-to-space fp32 NCHW (last decoder conv, sub-pixel form)
                        if (valid) {
                            const size_t plane = static_cast<size_t>(p.out_h) * p.out_w;
#pragma unroll
                            for (int j = 0; j < 16; ++j) {
                                const int ch = nb + j;
                                if (ch < p.c_out) {
                                    const int par = ch / p.shuffle_c, o = ch % p.shuffle_c;
                                    p.out32[(static_cast<size_t>(img) * p.shuffle_c + o) * plane +
                                            static_cast<size_t>(2 * Y + par / 2) * p.out_w + 2 * X + par % 2] =
                                        fmaf(__uint_as_float(v[j]), hscale, off[j]);
                                }
                            }
                        }
                    } else if (EPI == kEpiF32) {
                        // fp32 NCHW output (denoiser head: eps feeds the fp32 sampler)
                        if (valid) {
                            const size_t plane = static_cast<size_t>(p.out_h) * p.out_w;
                            float* o32 = p.out32 + (static_cast<size_t>(img) * p.c_out) * plane +
                                         static_cast<size_t>(oy) * p.out_w + ox;
#pragma unroll
                            for (int j = 0; j < 16; ++j) {
                                if (nb + j < p.c_out) {
                                    float a = fmaf(__uint_as_float(v[j]), hscale, off[j]);
                                    if (p.silu) a = silu_fast(a);
                                    o32[static_cast<size_t>(nb + j) * plane] = a;
                                }
                            }
                        }
                    } else if (p.tma_out || (valid && nb < p.cs_out)) {
                        __align__(16) __half2 h[8];
#pragma unroll
                        for (int j = 0; j < 16; j += 2) {
                            float a = fmaf(__uint_as_float(v[j]), hscale, off[j]);
                            float b = fmaf(__uint_as_float(v[j + 1]), hscale, off[j + 1]);
                            if (EPI == kEpiF16Silu) {
                                if (p.silu == 2) {
                                    a = silu_exact_h(a);
                                    b = silu_exact_h(b);
                                } else {
                                    a = fmaf(a, tanh_approx(a), a);
                                    b = fmaf(b, tanh_approx(b), b);
                                }
                            }
                            h[j / 2] = __floats2half2_rn(a, b);
                        }
                        if (p.tma_out) {
                            // 32 B rows, SWIZZLE_32B (tmO): 16-byte unit u of row r sits at u ^ (r / 4 % 2)
                            const uint32_t sb = stage_out_s + static_cast<uint32_t>(((warp - 2) * slots + (ring ? (stage_it & 1) : hh)) * schunk + lane * 32);
                            const uint32_t sw = ((sb >> 7) & 1u) << 4;  // address bit 7 (= lane / 4 % 2)
                            sts128u(sb + sw, *reinterpret_cast<uint4*>(&h[0]));
                            sts128u(sb + (16u ^ sw), *reinterpret_cast<uint4*>(&h[4]));
                        } else {
                            __half* dst =
                                p.out + ((static_cast<size_t>(img) * p.out_h + oy) * p.out_w + ox) * p.cs_out + nb;
                            uint4* d4 = reinterpret_cast<uint4*>(dst);
                            d4[0] = *reinterpret_cast<uint4*>(&h[0]);
                            d4[1] = *reinterpret_cast<uint4*>(&h[4]);
                        }
                    }
                }
                if (kTma && p.tma_out) {
                    // staged 32 px x 16 ch boxes -> global through the TMA unit
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0 && warp_store) {
                        const int nb0 = tc.n_tile * p.BN + c00;
                        const uint32_t sb = stage_out_s + static_cast<uint32_t>(((warp - 2) * slots + (ring ? (stage_it & 1) : 0)) * schunk);
                        if (p.planar32) {
                            if (nb0 < p.cs_out) tma_store_4d(&p.tmO[tc.parity], sb, bx, by, bi, nb0);
                            if (two && nb0 + kPair < p.cs_out)
                                tma_store_4d(&p.tmO[tc.parity], sb + schunk, bx, by, bi, nb0 + kPair);
                        } else {
                            if (nb0 < p.cs_out) tma_store_4d(&p.tmO[tc.parity], sb, nb0, bx, by, bi);
                            if (two && nb0 + kPair < p.cs_out)
                                tma_store_4d(&p.tmO[tc.parity], sb + schunk, nb0 + kPair, bx, by, bi);
                        }
                        bulk_commit();
                    }
                    ++stage_it;
                }
            }
            // release the accumulator buffer to the MMA warp (the leader's barrier)
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (CG == 1) mbar_arrive(&tempty[acc]);
                else mbar_arrive_cluster(acc ? tempty_leader1 : tempty_leader0);
            }
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
            if (next_switch) {
                cur ^= 1;
                cur_key = next_key;
                pending = true;
            }
        }
        if ((EPI <= kEpiF16Silu || EPI == kEpiF32Raw) && p.tma_out && lane == 0) bulk_wait0();
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

// Per-device caches (kernel attributes and SM counts apply per device; a
// process may drive several contexts on different GPUs).
constexpr int kMaxDevices = 64;
int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev < 0 || dev >= kMaxDevices ? 0 : dev;
}

int sm_count() {
    static int n[kMaxDevices] = {};
    const int dev = current_device();
    if (!n[dev]) {
        cudaDeviceGetAttribute(&n[dev], cudaDevAttrMultiProcessorCount, dev);
        if (n[dev] <= 0) n[dev] = 148;
    }
    return n[dev];
}

template <int CG>
size_t smem_bytes_for(const ConvParams& p) {
    const int tabf = tab_floats(p.rc, p.BN);
    int total_kb = 0;
    for (int s = 0; s < p.nseg; ++s) total_kb += p.seg[s].ntaps * p.seg[s].ncb;
    const int b_res = CG == 1 && p.b_res;
    const int a_stage = a_stage_bytes(p);
    const size_t bblk = static_cast<size_t>(p.BN / CG) * kBK * 2;
    if (p.halo && !b_res)
        return kSmemFixed + static_cast<size_t>(kHaloAStages) * a_stage +
               static_cast<size_t>(halo_ring_bstages<CG>(p.BN, tabf, p.tma_out, p.nhwc32, a_stage)) * bblk +
               epi_smem_bytes(tabf, p.tma_out, p.nhwc32, 0);
    const int st = num_stages<CG>(p.BN, tabf, p.tma_out, b_res, total_kb, p.nhwc32, a_stage);
    return kSmemFixed + static_cast<size_t>(st) * (a_stage + (b_res ? 0 : bblk)) + (b_res ? total_kb * bblk : 0) +
           epi_smem_bytes(tabf, p.tma_out, p.nhwc32, b_res);
}

int g_cta_group_override = -1;  // LC_CTA_GROUP env: 1 or 2 forces the variant

template <int CG, int EPI>
cudaError_t launch_variant(const ConvParams& p0, int parities, cudaStream_t stream) {
    ConvParams p = p0;
    {
        const int m_tiles = p.tiles_x * p.tiles_y * p.tiles_i;
        p.fd_units.init(static_cast<uint32_t>((m_tiles + CG - 1) / CG));
        p.fd_ntiles.init(static_cast<uint32_t>(p.n_pad / p.BN));
        p.fd_par.init(static_cast<uint32_t>(p.nparity));
        p.fd_tx.init(static_cast<uint32_t>(p.tiles_x));
        p.fd_ty.init(static_cast<uint32_t>(p.tiles_y));
    }
    // BN / 16 chunks over kEpiGroups warps per lane quarter leave some warps
    // one chunk more per tile (BN 160: 3, 3, 2, 2); rotating the assignment
    // by BN/16 mod kEpiGroups each tile evens the load over consecutive
    // tiles (two accumulators of slack)
    static const int rot_env = std::getenv("LC_EPI_ROT") ? std::atoi(std::getenv("LC_EPI_ROT")) : 1;
    p.epi_rot = rot_env ? (p.BN / 16) % kEpiGroups : 0;
    static bool attr_set[kMaxDevices] = {};
    const int dev = current_device();
    if (!attr_set[dev]) {
        cudaError_t e =
            cudaFuncSetAttribute(conv_tc_kernel<CG, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax);
        if (e != cudaSuccess) return e;
        attr_set[dev] = true;
    }
    const int n_tiles = p.n_pad / p.BN;
    const int m_tiles = p.tiles_x * p.tiles_y * p.tiles_i;
    if (CG == 1) {
        const int total = m_tiles * n_tiles * parities;
        int grid = total < sm_count() ? total : sm_count();
        if (p.b_res) grid = (sm_count() / (n_tiles * parities)) * n_tiles * parities;
        return launch_pdl(conv_tc_kernel<1, EPI>, dim3(grid), dim3(kThreads), smem_bytes_for<1>(p), stream, p,
                          n_tiles, parities);
    }
    const int units = ((m_tiles + 1) / 2) * n_tiles * parities;
    const int pairs = units < sm_count() / 2 ? units : sm_count() / 2;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem_bytes_for<2>(p);
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, conv_tc_kernel<CG, EPI>, p, n_tiles, parities);
}

template <int CG>
cudaError_t launch_cg(const ConvParams& p, int parities, cudaStream_t stream) {
    if (p.out32) {
        if (p.nhwc32) return launch_variant<CG, kEpiF32Raw>(p, parities, stream);
        if (p.shuffle_c > 0) return launch_variant<CG, kEpiShuffle>(p, parities, stream);
        return launch_variant<CG, kEpiF32>(p, parities, stream);
    }
    if (p.silu) return launch_variant<CG, kEpiF16Silu>(p, parities, stream);
    return launch_variant<CG, kEpiF16>(p, parities, stream);
}

}  // namespace

size_t conv_tc_smem_bytes(const ConvParams& p) {
    return p.cg == 2 ? smem_bytes_for<2>(p) : smem_bytes_for<1>(p);
}

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
    // A long K loop (>= 64 blocks) also takes pairs when they fill >= 3/4 of
    // the pair slots in one wave: single CTAs are ~35 % slower per tile there
    // (B's mid block: 144 single CTAs of BN 144 -> 64 pairs of BN 160).
    const bool ok = BN % 32 == 0 && m_tiles >= 2;
    const int pair_units = (m_tiles + 1) / 2 * n_tiles * parities;
    int cg = (ok && k_blocks >= 32 &&
              (m_tiles * n_tiles * parities >= 2 * sm_count() || (k_blocks >= 64 && 4 * pair_units >= 3 * (sm_count() / 2))))
                 ? 2
                 : 1;
    if (g_cta_group_override == 1) cg = 1;
    if (g_cta_group_override == 2 && ok) cg = 2;
    return cg;
}

// Weight-stationary schedule when it pays: one CTA group per (parity, N
// tile) slab, several M tiles per CTA, and the slab's weight panel plus >= 3
// activation stages fit in shared memory.  LC_BRES=0 disables it.
static bool want_b_res(const ConvParams& p, int parities) {
    static const int env = std::getenv("LC_BRES") ? std::atoi(std::getenv("LC_BRES")) : 1;
    if (!env || p.cg != 1) return false;
    const int n_tiles = p.n_pad / p.BN, slabs = n_tiles * parities;
    const int m_tiles = p.tiles_x * p.tiles_y * p.tiles_i;
    if (slabs > sm_count()) return false;
    const int cps = sm_count() / slabs;
    if (m_tiles < 2 * cps) return false;
    int total_kb = 0;
    for (int s = 0; s < p.nseg; ++s) total_kb += p.seg[s].ntaps * p.seg[s].ncb;
    // >= 3 activation stages; >= 2 halo stages (each carries every tap of a channel block)
    const int a_stage = a_stage_bytes(p), min_stages = p.halo ? 2 : 3;
    return num_stages<1>(p.BN, tab_floats(p.rc, p.BN), p.tma_out, 1, total_kb, p.nhwc32, a_stage) >= min_stages &&
           (kSmemMax - kSmemFixed - epi_smem_bytes(tab_floats(p.rc, p.BN), p.tma_out, p.nhwc32, 1) -
            total_kb * p.BN * kBK * 2) >= min_stages * a_stage;
}

static bool halo_ring_fits(const ConvParams& p) {
    const int tabf = tab_floats(p.rc, p.BN), a_stage = a_stage_bytes(p);
    return (p.cg == 2 ? halo_ring_bstages<2>(p.BN, tabf, p.tma_out, p.nhwc32, a_stage)
                      : halo_ring_bstages<1>(p.BN, tabf, p.tma_out, p.nhwc32, a_stage)) > 0;
}

bool conv_tc_halo_fits(const ConvParams& p, int parities) {
    if (!p.halo || p.nseg != 1) return false;
    if (p.cg == 1 && want_b_res(p, parities)) return true;
    static const int ring = std::getenv("LC_HALO_RING") ? std::atoi(std::getenv("LC_HALO_RING")) : 1;
    return ring && halo_ring_fits(p);
}

cudaError_t launch_conv_tc(const ConvParams& p, int parities, cudaStream_t stream) {
    if (p.halo) {
        // weight-stationary when it pays (as below), else halo + weight rings
        if (!conv_tc_halo_fits(p, parities)) return cudaErrorInvalidValue;
        ConvParams q = p;
        q.b_res = p.cg == 1 && want_b_res(p, parities) ? 1 : 0;
        return p.cg == 2 ? launch_cg<2>(q, parities, stream) : launch_cg<1>(q, parities, stream);
    }
    if (p.cg == 2) return launch_cg<2>(p, parities, stream);
    if (want_b_res(p, parities)) {
        ConvParams q = p;
        q.b_res = 1;
        return launch_cg<1>(q, parities, stream);
    }
    return launch_cg<1>(p, parities, stream);
}

}  // namespace lc
