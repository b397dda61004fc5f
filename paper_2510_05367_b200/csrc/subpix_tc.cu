// K8: fused tap-to-N convolutions (see subpix_tc.cuh).
//
// Tile: 5 x 64 pixels of one image (low-res pixels for the decoder).  The
// TMA box stages the 7 x 66 window around it (out-of-image pixels are
// zero-filled); its 462 pixels, flattened row-major, are the M rows (4
// M-tiles of 128) of the GEMM y = window x tapbank^T, fp32 in TMEM.  Then
//   decoder: out(2Y+py, 2X+px) = bias + sum_{t=(dy,dx)} y[(Y+dy-1+py, X+dx-1+px)][(p*4+t)*C + c]
//   head:    out(Y, X) = sum_{in-window taps} s*y[(Y+ky-1, X+kx-1)][t*C + c]
//                        + o * sum_{in-window taps} wsum[t][c] + bias[c]
// -- the sums, in the order, of the tap-to-N GEMM + gather kernel pairs
// these replace (kernels.cu tap_gather_kernel / subpix_gather_kernel).
//
// Warps: 0 TMA producer, 1 MMA issuer (+ TMEM owner), 2..9 epilogue.  Two
// A stages (one 64-channel K block each) and two TMEM accumulators, so the
// loads and MMAs of tile i+1 run under the epilogue of tile i.  Epilogue per
// tile: all tap columns of every staged pixel TMEM -> shared (the
// accumulator is released right after), barrier, gather + coalesced planar
// stores (decoder: both column parities of an output row as one float2),
// barrier.  A first version with one epilogue pass per output parity (four
// barrier pairs per tile, bias/wsum re-read per output) ran the decoder
// stage at 6.9 us per tile, 22 % of HBM bandwidth; a third A stage did not
// change that.
#include "subpix_tc.cuh"

#include <cstdlib>

#include "pdl.cuh"
#include "ptx.cuh"

namespace lc {

namespace {

// Per mode: staged pixels, M-tiles of 128, A stage stride.  The MMA of the
// last M-tile reads past the staged rows into the next stage (or the tap
// bank): those rows only feed accumulator rows that are never read.
template <int MODE, int TYV> struct Geo {
    static constexpr int TY = TYV, SY = TYV + 2;
    static constexpr int NPix = kTapSX * SY;                   // staged pixels (decoder TY 5: 462)
    // GEMM rows: the head multiplies every staged pixel; the decoder only
    // the TY output rows of the window (its row taps are summed inside the
    // MMA through row-shifted A descriptors, see the kernel)
    static constexpr int MRows = MODE == kTapSubpix ? kTapSX * TY : NPix;
    static constexpr int MT = (MRows + 127) / 128;
    static constexpr int ABytes = (NPix * 128 + 1023) / 1024 * 1024;
    static constexpr int KRep = MODE == kTapSubpix ? 3 : 1;    // weight K blocks per input K block
    // A ring depth: shorter decoder tiles buy more stages in flight
    static constexpr int ST = MODE == kTapSubpix ? (TY <= 3 ? 4 : TY == 4 ? 3 : 2) : (TY <= 3 ? 3 : 2);
};
constexpr int kMaxPC = 36;  // tap columns per GEMM row (decoder 8*4, head 9*4)
constexpr int kEpiWarps = 8;
constexpr int kThreads = 32 * (2 + kEpiWarps);
constexpr int kAccCols = 256;                    // TMEM columns per accumulator buffer
constexpr int kSmemMax = 232448;

// shared-memory row stride (floats) of one staged pixel's pass columns:
// a multiple of 4 whose lane stride spreads 8 consecutive lanes' 16-byte
// stores over distinct bank quads
__host__ __device__ constexpr int y_stride(int mode, int C) {
    return mode == kTapSubpix ? (C == 1 ? 12 : C == 2 ? 20 : C == 3 ? 28 : 36) : (C == 1 ? 12 : C == 2 ? 20 : C == 3 ? 28 : 36);
}
// columns per GEMM row: decoder (py, px, dx, c) after the MMA summed dy; head (tap, c)
__host__ __device__ constexpr int pass_cols(int mode, int C) { return mode == kTapSubpix ? 8 * C : 9 * C; }
// the fused sampler step keeps e_u of one tile: C x TY x TX floats
template <int MODE, int TY>
constexpr int eu_bytes() {
    return MODE == kTapConv3 ? 4 * TY * kTapTX * 4 : 0;
}
template <int MODE, int TY>
int smem_bytes(const TapTcParams& p) {
    using G = Geo<MODE, TY>;
    return 1024 + G::ST * G::ABytes + G::KRep * p.kb * p.N * 128 + G::MRows * y_stride(MODE, p.C) * 4 +
           eu_bytes<MODE, TY>() + 512;
}

__device__ __forceinline__ void tmem_ld4(uint32_t taddr, uint32_t (&v)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "r"(taddr));
}

template <int MODE, int TYV>
__global__ void __launch_bounds__(kThreads, 1) tap_tc_kernel(const __grid_constant__ TapTcParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    using G = Geo<MODE, TYV>;
    constexpr int kNPix = G::NPix, kMT = G::MT, kABytes = G::ABytes;
    constexpr int kMRows = G::MRows, kKRep = G::KRep, kStages = G::ST;
    constexpr int kTapTY = G::TY;
    const int C = p.C, N = p.N, YS = y_stride(MODE, C), PC = pass_cols(MODE, C);
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* smA = smem;
    uint8_t* smW = smA + kStages * kABytes;
    float* smY = reinterpret_cast<float*>(smW + kKRep * p.kb * N * 128);
    float* smEu = smY + kMRows * YS;  // [C][TY][TX] e_u of the pair's first tile (head, pair_T > 0)
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(smEu) + eu_bytes<MODE, TYV>());
    uint64_t* full_bar = bars;                  // [kStages]
    uint64_t* empty_bar = bars + kStages;       // [kStages]
    uint64_t* tfull = bars + 2 * kStages;       // [2]
    uint64_t* tempty = bars + 2 * kStages + 2;  // [2]
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 4);
    float* sm_bias = reinterpret_cast<float*>(bars + 2 * kStages + 6);  // [4]
    float* sm_wsum = sm_bias + 4;                                       // [9][C]

    const int warp = __shfl_sync(0xffffffff, static_cast<int>(threadIdx.x) / 32, 0);
    const int lane = static_cast<int>(threadIdx.x) & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], kEpiWarps);
        }
        fence_barrier_init();
    }
    if (warp == 0 && lane == 0) tma_prefetch_desc(&p.tmA);
    if (warp == 1) tmem_alloc<512>(tmem_holder);
    // tap bank -> shared, K-major rows of 128 B in the 128B-swizzle layout
    // the MMA descriptor expects (16 B chunk j of row r at j ^ (r & 7))
    {
        const int wkb = kKRep * p.kb;  // decoder: K blocks ordered (row offset o, channel block)
        const int chunks = wkb * N * 8;
        for (int i = static_cast<int>(threadIdx.x); i < chunks; i += kThreads) {
            const int k = i / (N * 8), r = (i / 8) % N, j = i % 8;
            const uint4 v = *reinterpret_cast<const uint4*>(p.w + static_cast<size_t>(r) * (wkb * 64) + k * 64 + j * 8);
            sts128u(smem_u32(smW + k * N * 128 + r * 128 + ((j ^ (r & 7)) << 4)), v);
        }
        fence_proxy_async_smem();
        if (threadIdx.x < 4) sm_bias[threadIdx.x] = static_cast<int>(threadIdx.x) < C ? p.bias[threadIdx.x] : 0.f;
        if (MODE == kTapConv3 && static_cast<int>(threadIdx.x) < 9 * C) sm_wsum[threadIdx.x] = p.wsum[threadIdx.x];
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    pdl_trigger();
    pdl_wait();

    const int tiles_per_img = p.tiles_x * p.tiles_y;
    auto tile_origin = [&](int tile, int& n, int& Y0, int& X0) {
        n = tile / tiles_per_img;
        const int r = tile - n * tiles_per_img;
        const int ty = r / p.tiles_x;
        Y0 = p.win.oy0 + ty * kTapTY;
        X0 = p.win.ox0 + (r - ty * p.tiles_x) * kTapTX;
    };
    // The CTA's k-th tile (-1: done).  Fused sampler step: unit u = (frame,
    // tile) of the uncond branch, its two images' tiles back to back.
    const bool paired = MODE == kTapConv3 && p.pair_T > 0;
    auto tile_at = [&](int k) -> int {
        if (!paired) {
            const int t = static_cast<int>(blockIdx.x) + k * static_cast<int>(gridDim.x);
            return t < p.num_tiles ? t : -1;
        }
        const int u = static_cast<int>(blockIdx.x) + (k >> 1) * static_cast<int>(gridDim.x);
        if (u >= p.pair_T * tiles_per_img) return -1;
        return u + (k & 1) * p.pair_T * tiles_per_img;
    };

    if (warp == 0) {
        // ------------------------------------------------------ TMA producer
        if (elect_one()) {
            int it = 0;
            for (int kt = 0, tile; (tile = tile_at(kt)) >= 0; ++kt) {
                int n, Y0, X0;
                tile_origin(tile, n, Y0, X0);
                for (int k = 0; k < p.kb; ++k, ++it) {
                    const int s = it % kStages;
                    mbar_wait(&empty_bar[s], ((it / kStages) & 1) ^ 1);
                    mbar_arrive_expect_tx(&full_bar[s], kNPix * 128);
                    tma_load_4d(smA + s * kABytes, &p.tmA, &full_bar[s], k * 64, X0 - 1, Y0 - 1, n);
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------ MMA issuer
        const uint32_t idesc = umma_idesc_f16(128, static_cast<uint32_t>(N));
        int it = 0, lt = 0;
        for (; tile_at(lt) >= 0; ++lt) {
            const int buf = lt & 1;
            mbar_wait(&tempty[buf], ((lt >> 1) & 1) ^ 1);
            tc_fence_after();
            const uint32_t d0 = tmem_base + buf * kAccCols;
            for (int k = 0; k < p.kb; ++k, ++it) {
                const int s = it % kStages;
                mbar_wait(&full_bar[s], (it / kStages) & 1);
                tc_fence_after();
                if (elect_one()) {
                    // decoder: one pass per window-row offset o of the output
                    // rows' taps (dy + py), its A rows shifted by o image rows
                    // (a 128 B-row start-address shift of the SW128 tile, see
                    // conv_tc.cu halo staging); the head: o = 0 only
#pragma unroll
                    for (int o = 0; o < kKRep; ++o) {
                        const uint64_t bdesc = umma_desc_sw128(smem_u32(smW + (o * p.kb + k) * N * 128));
#pragma unroll
                        for (int mt = 0; mt < kMT; ++mt) {
                            const uint64_t adesc =
                                umma_desc_sw128(smem_u32(smA + s * kABytes + (mt * 128 + o * kTapSX) * 128));
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk)
                                umma_f16(d0 + mt * N, adesc + 2 * kk, bdesc + 2 * kk, idesc,
                                         (k | o | kk) != 0 ? 1u : 0u);
                        }
                    }
                    umma_commit(&empty_bar[s]);
                }
                __syncwarp();
            }
            if (elect_one()) umma_commit(&tfull[buf]);
            __syncwarp();
        }
    } else {
        // ------------------------------------------------------ epilogue
        const int e = warp - 2;                 // 0..7
        const int qd = warp & 3;                // TMEM lane quarter this warp may read
        const int g = e >> 2;                   // M-tiles g, g+2
        const int et = static_cast<int>(threadIdx.x) - 64;
        const uint32_t ybase = smem_u32(smY);
        const float yscale = p.scale;
        const int nld = (PC + 3) / 4;
        const int OH = MODE == kTapSubpix ? 2 * p.H : p.H, OW = MODE == kTapSubpix ? 2 * p.W : p.W;
        const size_t plane = static_cast<size_t>(OH) * OW;
        constexpr int kTilePx = kTapTY * kTapTX;
        // i / C as a multiply-high (exact for i < 2^31, C <= 4; C == 1 separately)
        const uint32_t cmag = C > 1 ? 0xFFFFFFFFu / static_cast<uint32_t>(C) + 1u : 0u;
        int lt = 0;
        int bad = 0;
        for (int tile; (tile = tile_at(lt)) >= 0; ++lt) {
            const int buf = lt & 1;
            int n, Y0, X0;
            tile_origin(tile, n, Y0, X0);
            mbar_wait(&tfull[buf], (lt >> 1) & 1);
            tc_fence_after();
            // every staged pixel's tap columns -> shared (all loads in flight, one wait)
            for (int mt = g; mt < kMT; mt += 2) {
                const int q = mt * 128 + qd * 32 + lane;
                const uint32_t ta = tmem_base + (static_cast<uint32_t>(qd * 32) << 16) +
                                    static_cast<uint32_t>(buf * kAccCols + mt * N);
                uint32_t v[kMaxPC];
#pragma unroll
                for (int j = 0; j < kMaxPC / 4; ++j)
                    if (j < nld) tmem_ld4(ta + 4 * j, *reinterpret_cast<uint32_t(*)[4]>(&v[4 * j]));
                tmem_ld_wait();
                if (q < kMRows) {
#pragma unroll
                    for (int j = 0; j < kMaxPC / 4; ++j)
                        if (j < nld)
                            sts128(ybase + static_cast<uint32_t>((q * YS + 4 * j) * 4),
                                   make_float4(__uint_as_float(v[4 * j]) * yscale, __uint_as_float(v[4 * j + 1]) * yscale,
                                               __uint_as_float(v[4 * j + 2]) * yscale,
                                               __uint_as_float(v[4 * j + 3]) * yscale));
                }
            }
            // the accumulator is in shared memory now: release it to the MMA warp
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[buf]);
            named_bar_sync(1, 32 * kEpiWarps);
            if (MODE == kTapSubpix) {
                // task (c, py, ry, rx): out(2Y+py, 2X+px) = bias + sum_dx y[(ry, rx+px+dx)][((py*2+px)*2+dx)*C + c]
                // (the row taps dy are already summed by the MMA)
                for (int i = et; i < kTilePx * 2 * C; i += 32 * kEpiWarps) {
                    int c, r;
                    if (p.cfast) {
                        r = C == 1 ? i : static_cast<int>(__umulhi(static_cast<uint32_t>(i), cmag));
                        c = i - r * C;
                    } else {
                        c = i / (2 * kTilePx);
                        r = i - c * 2 * kTilePx;
                    }
                    const int py = r / kTilePx, r2 = r - py * kTilePx;
                    const int ry = r2 / kTapTX, rx = r2 - ry * kTapTX;
                    const int Y = Y0 + ry, X = X0 + rx;
                    if (Y >= p.win.oy1 || X >= p.win.ox1) continue;
                    float o2[2];
#pragma unroll
                    for (int px = 0; px < 2; ++px) {
                        const int q = ry * kTapSX + rx + px;
                        const int col = ((py * 2 + px) * 2) * C + c;
                        o2[px] = sm_bias[c] + smY[q * YS + col] + smY[(q + 1) * YS + col + C];
                    }
                    *reinterpret_cast<float2*>(p.out + (static_cast<size_t>(n) * C + c) * plane +
                                               static_cast<size_t>(2 * Y + py) * OW + 2 * X) = make_float2(o2[0], o2[1]);
                }
            } else {
                // task (c, ry, rx): out(Y, X) = sum_in s*y + (o * sum_in wsum + bias)
                for (int i = et; i < kTilePx * C; i += 32 * kEpiWarps) {
                    int c, r;
                    if (p.cfast) {
                        r = C == 1 ? i : static_cast<int>(__umulhi(static_cast<uint32_t>(i), cmag));
                        c = i - r * C;
                    } else {
                        c = i / kTilePx;
                        r = i - c * kTilePx;
                    }
                    const int ry = r / kTapTX, rx = r - ry * kTapTX;
                    const int Y = Y0 + ry, X = X0 + rx;
                    if (Y >= p.win.oy1 || X >= p.win.ox1) continue;
                    float acc = 0.f, ws = 0.f;
#pragma unroll
                    for (int ky = 0; ky < 3; ++ky) {
                        const int sy = Y + ky - 1;
                        const bool rin = sy >= p.win.vy0 && sy < p.win.vy1;
#pragma unroll
                        for (int kx = 0; kx < 3; ++kx) {
                            const int sx = X + kx - 1;
                            const bool in = rin && sx >= p.win.vx0 && sx < p.win.vx1;
                            const int t = ky * 3 + kx;
                            const float v = smY[((ry + ky) * kTapSX + rx + kx) * YS + t * C + c];
                            acc += in ? v : 0.f;
                            ws += in ? sm_wsum[t * C + c] : 0.f;
                        }
                    }
                    const float e = acc + fmaf(p.shift, ws, sm_bias[c]);
                    if (!paired) {
                        p.out[(static_cast<size_t>(n) * C + c) * plane + static_cast<size_t>(Y) * OW + X] = e;
                    } else if (lt & 1) {
                        // cond branch: cfg_combine then the sampler update
                        const float eu = smEu[i];
                        const float eps = __fadd_rn(__fmul_rn(1.0f - p.g, eu), __fmul_rn(p.g, e));
                        const size_t xi = (static_cast<size_t>(n - p.pair_T) * C + c) * plane +
                                          static_cast<size_t>(Y) * OW + X;
                        float xn = __fadd_rn(__fmul_rn(p.a, p.x[xi]), __fmul_rn(p.b, eps));
                        if (p.z) xn = __fadd_rn(__fmul_rn(1.0f, xn), __fmul_rn(p.c, p.z[xi]));
                        p.x_out[xi] = xn;
                        bad |= !isfinite(xn);
                    } else {
                        smEu[i] = e;  // uncond branch: kept for the pair's second tile
                    }
                }
            }
            named_bar_sync(1, 32 * kEpiWarps);  // shared y is rewritten by the next tile
        }
        // one flag write per warp (warp-wide vote)
        if (paired && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(p.bad, 1);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<512>(tmem_base);
    }
}

template <int MODE, int TY>
cudaError_t launch_mode(const TapTcParams& p, cudaStream_t st) {
    // per device: the attribute applies to the current device only
    constexpr int kMaxDevices = 64;
    static bool attr[kMaxDevices] = {};
    static int sm[kMaxDevices] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDevices) dev = 0;
    if (!attr[dev]) {
        const cudaError_t e =
            cudaFuncSetAttribute(tap_tc_kernel<MODE, TY>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax);
        if (e != cudaSuccess) return e;
        attr[dev] = true;
    }
    if (!sm[dev]) {
        cudaDeviceGetAttribute(&sm[dev], cudaDevAttrMultiProcessorCount, dev);
        if (sm[dev] <= 0) sm[dev] = 148;
    }
    const int sms = sm[dev];
    const int units = (MODE == kTapConv3 && p.pair_T > 0) ? p.pair_T * p.tiles_x * p.tiles_y : p.num_tiles;
    const int grid = units < sms ? units : sms;
    // LC_TAP_CFAST=1: channel-fastest epilogue tasks, so a warp's 32 reads of
    // the staged tap columns cover 32 / C pixels x C channels in distinct
    // banks (the pixel-fastest order strides by the 28 / 36-float row: 4-way
    // conflicts).  8x fewer conflicts, same kernel time: off.
    static const int cfast = std::getenv("LC_TAP_CFAST") ? std::atoi(std::getenv("LC_TAP_CFAST")) : 0;
    TapTcParams q = p;
    q.cfast = cfast;
    return launch_pdl(tap_tc_kernel<MODE, TY>, dim3(grid), dim3(kThreads), static_cast<size_t>(smem_bytes<MODE, TY>(p)),
                      st, q);
}

template <int MODE, int TY>
bool fits(int C, int kb, int N) {
    TapTcParams p{};
    p.C = C;
    p.kb = kb;
    p.N = N;
    return C >= 1 && C <= 4 && kb >= 1 && kb <= kTapMaxKb && N % 16 == 0 && N >= pass_cols(MODE, C) &&
           pass_cols(MODE, C) <= kMaxPC && Geo<MODE, TY>::MT * N <= kAccCols && smem_bytes<MODE, TY>(p) <= kSmemMax;
}

}  // namespace

// Decoder tile height: TY 5 with a 2-stage A ring by default; LC_K8_TY = 3 /
// 4 (4 / 3 stages) for A/B timing.  Measured on D (one box, back to back):
// 26.95k / 26.66k / 26.73k frames/s for TY 3 / 4 / 5 -- the deeper rings buy
// nothing once the row taps are summed in the MMA (the epilogue then waits
// on the MMA: 72 N = 32 instructions per tile, tensor pipe 59 % active).
int tap_tile_rows(int mode, int C, int kb, int N) {
    if (mode != kTapSubpix) {
        // head: TY 5 (2 stages) by default; LC_K8_HEAD_TY=3 (3 stages) for A/B timing
        static const int henv = std::getenv("LC_K8_HEAD_TY") ? std::atoi(std::getenv("LC_K8_HEAD_TY")) : 5;
        return henv == 3 && fits<kTapConv3, 3>(C, kb, N) ? 3 : 5;
    }
    static const int env = std::getenv("LC_K8_TY") ? std::atoi(std::getenv("LC_K8_TY")) : 5;
    if (env == 3 && fits<kTapSubpix, 3>(C, kb, N)) return 3;
    if (env == 4 && fits<kTapSubpix, 4>(C, kb, N)) return 4;
    return 5;
}

bool tap_tc_supported(int mode, int C, int kb, int N) {
    if (mode != kTapSubpix)
        return tap_tile_rows(mode, C, kb, N) == 3 ? fits<kTapConv3, 3>(C, kb, N) : fits<kTapConv3, 5>(C, kb, N);
    switch (tap_tile_rows(mode, C, kb, N)) {
        case 3: return fits<kTapSubpix, 3>(C, kb, N);
        case 4: return fits<kTapSubpix, 4>(C, kb, N);
        default: return fits<kTapSubpix, 5>(C, kb, N);
    }
}

cudaError_t launch_tap_tc(int mode, const TapTcParams& p, cudaStream_t st) {
    if (!tap_tc_supported(mode, p.C, p.kb, p.N)) return cudaErrorInvalidValue;
    if (p.num_tiles <= 0) return cudaSuccess;
    if (mode == kTapConv3)
        return tap_tile_rows(mode, p.C, p.kb, p.N) == 3 ? launch_mode<kTapConv3, 3>(p, st) : launch_mode<kTapConv3, 5>(p, st);
    switch (tap_tile_rows(mode, p.C, p.kb, p.N)) {
        case 3: return launch_mode<kTapSubpix, 3>(p, st);
        case 4: return launch_mode<kTapSubpix, 4>(p, st);
        default: return launch_mode<kTapSubpix, 5>(p, st);
    }
}

}  // namespace lc
