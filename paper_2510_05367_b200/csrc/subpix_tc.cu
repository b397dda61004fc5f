// K8: fused last decoder stage (see subpix_tc.cuh).
//
// Tile: kSubpixTY x kSubpixTX low-res pixels of one frame.  The TMA box
// stages the (TY+2) x (TX+2) window around it (out-of-image pixels are
// zero-filled, which is the conv's zero padding); its pixels, flattened
// row-major, are the M rows of the GEMM y = window x tapbank^T (N = 16*C,
// K = c_in), 4 M-tiles of 128 (462 staged pixels), fp32 in TMEM.  Output
// pixel (2Y+py, 2X+px) = bias + sum over its 2x2 source taps t = (dy,dx) of
// y[pixel (Y+dy-1+py, X+dx-1+px)][(p*4+t)*C + c] -- the same sums, in the
// same order, as the tap-to-N GEMM + subpix_gather_kernel pair it replaces.
//
// Warps: 0 TMA producer, 1 MMA issuer (+ TMEM owner), 2..9 epilogue.  Two
// A stages (one 64-channel K block each) and two TMEM accumulators, so the
// loads and MMAs of tile i+1 run under the epilogue of tile i.  Epilogue per
// output parity: TMEM -> shared (the parity's 4*C columns of every staged
// pixel), barrier, gather + coalesced planar stores, barrier.
#include "subpix_tc.cuh"

#include "pdl.cuh"
#include "ptx.cuh"

namespace lc {

namespace {

constexpr int kNPix = kSubpixSX * kSubpixSY;     // 462 staged pixels
constexpr int kMT = (kNPix + 127) / 128;         // 4 M-tiles
constexpr int kABytes = kMT * 128 * 128;         // one A stage (64 channels x 512 rows)
constexpr int kStages = 2;
constexpr int kEpiWarps = 8;
constexpr int kThreads = 32 * (2 + kEpiWarps);
constexpr int kMaxKb = 4;
constexpr int kAccCols = 256;                    // TMEM columns per accumulator buffer

__host__ __device__ constexpr int y_stride(int C) { return C == 1 ? 4 : C == 4 ? 20 : 12; }

constexpr int kWBytesMax = kMaxKb * 64 * 128;
constexpr int kYBytesMax = kNPix * 20 * 4;
constexpr int kSmem = 1024 + kStages * kABytes + kWBytesMax + kYBytesMax + 256;

__device__ __forceinline__ void tmem_ld4(uint32_t taddr, uint32_t (&v)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "r"(taddr));
}

__global__ void __launch_bounds__(kThreads, 1) subpix_tc_kernel(const __grid_constant__ SubpixTcParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* smA = smem;
    uint8_t* smW = smA + kStages * kABytes;
    float* smY = reinterpret_cast<float*>(smW + kWBytesMax);
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(smY) + kYBytesMax);
    uint64_t* full_bar = bars;            // [kStages]
    uint64_t* empty_bar = bars + 2;       // [kStages]
    uint64_t* tfull = bars + 4;           // [2]
    uint64_t* tempty = bars + 6;          // [2]
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 8);

    const int warp = __shfl_sync(0xffffffff, static_cast<int>(threadIdx.x) / 32, 0);
    const int lane = static_cast<int>(threadIdx.x) & 31;
    const int C = p.C, N = 16 * C, YS = y_stride(C);

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
        const int chunks = p.kb * N * 8;
        for (int i = static_cast<int>(threadIdx.x); i < chunks; i += kThreads) {
            const int k = i / (N * 8), r = (i / 8) % N, j = i % 8;
            const uint4 v = *reinterpret_cast<const uint4*>(p.w + static_cast<size_t>(r) * (p.kb * 64) + k * 64 + j * 8);
            sts128u(smem_u32(smW + k * N * 128 + r * 128 + ((j ^ (r & 7)) << 4)), v);
        }
        fence_proxy_async_smem();
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
        Y0 = ty * kSubpixTY;
        X0 = (r - ty * p.tiles_x) * kSubpixTX;
    };

    if (warp == 0) {
        // ------------------------------------------------------ TMA producer
        if (elect_one()) {
            int it = 0;
            for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
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
        for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x, ++lt) {
            const int buf = lt & 1;
            mbar_wait(&tempty[buf], ((lt >> 1) & 1) ^ 1);
            tc_fence_after();
            const uint32_t d0 = tmem_base + buf * kAccCols;
            for (int k = 0; k < p.kb; ++k, ++it) {
                const int s = it % kStages;
                mbar_wait(&full_bar[s], (it / kStages) & 1);
                tc_fence_after();
                if (elect_one()) {
                    const uint64_t bdesc = umma_desc_sw128(smem_u32(smW + k * N * 128));
#pragma unroll
                    for (int mt = 0; mt < kMT; ++mt) {
                        const uint64_t adesc = umma_desc_sw128(smem_u32(smA + s * kABytes + mt * 128 * 128));
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            umma_f16(d0 + mt * N, adesc + 2 * kk, bdesc + 2 * kk, idesc, (k | kk) != 0 ? 1u : 0u);
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
        float bias[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) bias[c] = c < C ? __ldg(p.bias + c) : 0.f;
        const int H2 = 2 * p.H, W2 = 2 * p.W;
        const size_t plane = static_cast<size_t>(H2) * W2;
        int lt = 0;
        for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x, ++lt) {
            const int buf = lt & 1;
            int n, Y0, X0;
            tile_origin(tile, n, Y0, X0);
            mbar_wait(&tfull[buf], (lt >> 1) & 1);
            tc_fence_after();
            for (int par = 0; par < 4; ++par) {
                const int py = par >> 1, px = par & 1;
                // this parity's 4*C columns of every staged pixel -> shared
                for (int mt = g; mt < kMT; mt += 2) {
                    const int q = mt * 128 + qd * 32 + lane;
                    const uint32_t ta = tmem_base + (static_cast<uint32_t>(qd * 32) << 16) +
                                        static_cast<uint32_t>(buf * kAccCols + mt * N + par * 4 * C);
                    uint32_t v[16];
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (j < C) tmem_ld4(ta + 4 * j, *reinterpret_cast<uint32_t(*)[4]>(&v[4 * j]));
                    tmem_ld_wait();
                    if (q < kNPix) {
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            if (j < C)
                                sts128u(ybase + static_cast<uint32_t>((q * YS + 4 * j) * 4),
                                        make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]));
                    }
                }
                named_bar_sync(1, 32 * kEpiWarps);
                // gather: out(2Y+py, 2X+px) = bias + sum_t y[src(t)][t*C + c]
                for (int i = et; i < kSubpixTY * kSubpixTX; i += 32 * kEpiWarps) {
                    const int ry = i / kSubpixTX, rx = i - ry * kSubpixTX;
                    const int Y = Y0 + ry, X = X0 + rx;
                    if (Y >= p.H || X >= p.W) continue;
                    float acc[4];
#pragma unroll
                    for (int c = 0; c < 4; ++c) acc[c] = bias[c];
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const int q = (ry + (t >> 1) + py) * kSubpixSX + rx + (t & 1) + px;
                        const float* yp = smY + q * YS + t * C;
#pragma unroll
                        for (int c = 0; c < 4; ++c)
                            if (c < C) acc[c] += yp[c];
                    }
                    float* o = p.out + static_cast<size_t>(n) * C * plane + static_cast<size_t>(2 * Y + py) * W2 + 2 * X + px;
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        if (c < C) o[c * plane] = acc[c];
                }
                named_bar_sync(1, 32 * kEpiWarps);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[buf]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<512>(tmem_base);
    }
}

}  // namespace

cudaError_t launch_subpix_tc(const SubpixTcParams& p, cudaStream_t st) {
    if (p.C < 1 || p.C > 4 || p.kb < 1 || p.kb > kMaxKb) return cudaErrorInvalidValue;
    static bool attr = false;
    if (!attr) {
        const cudaError_t e = cudaFuncSetAttribute(subpix_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int grid = p.num_tiles < sms ? p.num_tiles : sms;
    return launch_pdl(subpix_tc_kernel, dim3(grid), dim3(kThreads), kSmem, st, p);
}

}  // namespace lc
