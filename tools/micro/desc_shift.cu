// Micro-test: can a tcgen05.mma A operand start at a row that is not a
// multiple of 8 inside a SWIZZLE_128B K-major tile (start address shifted by
// s * 128 B), and which descriptor base-offset value makes it correct?
// This decides whether a conv tile can feed several taps from ONE halo box
// (row-shifted descriptors) instead of one TMA box per tap.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2510_05367_b200/csrc \
//        tools/micro/desc_shift.cu -o gpurun_out/desc_shift && gpurun_out/desc_shift
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "ptx.cuh"

using namespace lc;

constexpr int kRows = 136, kN = 64, kK = 64, kShifts = 9, kVar = 3;

__device__ uint64_t desc(uint32_t saddr, uint32_t base_off) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
    d |= static_cast<uint64_t>(1) << 16;
    d |= static_cast<uint64_t>(1024 >> 4) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(base_off & 7) << 49;
    d |= static_cast<uint64_t>(2) << 61;
    return d;
}

__global__ void k(const __half* A, const __half* B, float* out) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = sm;                      // 136 rows x 128 B = 17 KB
    uint8_t* sB = sm + 18 * 1024;          // 64 rows x 128 B
    __shared__ uint64_t bar;
    __shared__ uint32_t holder;
    const int t = threadIdx.x;
    // SW128 as TMA writes it: 16 B chunk c of row r lands at chunk c ^ (r & 7)
    for (int e = t; e < kRows * 8; e += blockDim.x) {
        const int r = e / 8, c = e % 8;
        *reinterpret_cast<uint4*>(sA + r * 128 + ((c ^ (r & 7)) * 16)) =
            *reinterpret_cast<const uint4*>(A + r * kK + c * 8);
    }
    for (int e = t; e < kN * 8; e += blockDim.x) {
        const int r = e / 8, c = e % 8;
        *reinterpret_cast<uint4*>(sB + r * 128 + ((c ^ (r & 7)) * 16)) =
            *reinterpret_cast<const uint4*>(B + r * kK + c * 8);
    }
    if (t == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    if (t < 32) tmem_alloc<64>(&holder);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = holder;
    const uint32_t idesc = umma_idesc_f16(128, kN);
    uint32_t phase = 0;
    for (int s = 0; s < kShifts; ++s)
        for (int v = 0; v < kVar; ++v) {
            if (t == 0) {
                const uint32_t a0 = smem_u32(sA) + s * 128;
                const uint32_t bo = v == 0 ? 0u : v == 1 ? (s & 7) : ((8 - (s & 7)) & 7);
                const uint64_t ad = desc(a0, bo), bd = desc(smem_u32(sB), 0);
                for (int kk = 0; kk < kK / 16; ++kk) umma_f16(tm, ad + 2 * kk, bd + 2 * kk, idesc, kk != 0);
                umma_commit(&bar);
            }
            __syncwarp();
            mbar_wait(&bar, phase);
            phase ^= 1;
            tc_fence_after();
            const int w = t / 32, l = t % 32;
            for (int c0 = 0; c0 < kN; c0 += 16) {
                uint32_t r[16];
                tmem_ld16(tm + (static_cast<uint32_t>(w * 32) << 16) + c0, r);
                tmem_ld_wait();
                for (int j = 0; j < 16; ++j)
                    out[((s * kVar + v) * 128 + w * 32 + l) * kN + c0 + j] = __uint_as_float(r[j]);
            }
            tc_fence_before();
            __syncthreads();
            tc_fence_after();
        }
    if (t < 32) tmem_dealloc<64>(tm);
}

int main() {
    std::vector<__half> A(kRows * kK), B(kN * kK);
    std::vector<float> Af(A.size()), Bf(B.size());
    srand(1);
    for (size_t i = 0; i < A.size(); ++i) { A[i] = __float2half((rand() % 17 - 8) / 8.0f); Af[i] = __half2float(A[i]); }
    for (size_t i = 0; i < B.size(); ++i) { B[i] = __float2half((rand() % 17 - 8) / 8.0f); Bf[i] = __half2float(B[i]); }
    __half *dA, *dB;
    float* dO;
    const size_t on = static_cast<size_t>(kShifts) * kVar * 128 * kN;
    cudaMalloc(&dA, A.size() * 2);
    cudaMalloc(&dB, B.size() * 2);
    cudaMalloc(&dO, on * 4);
    cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
    k<<<1, 128, 40 * 1024>>>(dA, dB, dO);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<float> O(on);
    cudaMemcpy(O.data(), dO, on * 4, cudaMemcpyDeviceToHost);
    for (int s = 0; s < kShifts; ++s) {
        printf("shift %d:", s);
        for (int v = 0; v < kVar; ++v) {
            double err = 0;
            for (int m = 0; m < 128; ++m)
                for (int n = 0; n < kN; ++n) {
                    double ref = 0;
                    for (int kk = 0; kk < kK; ++kk) ref += Af[(s + m) * kK + kk] * Bf[n * kK + kk];
                    err = fmax(err, fabs(ref - O[((s * kVar + v) * 128 + m) * kN + n]));
                }
            printf("  var%d maxerr %.3g", v, err);
        }
        printf("\n");
    }
    return 0;
}
