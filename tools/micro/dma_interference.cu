// Microbenchmark: does a concurrent host-link DMA slow a write-heavy or a
// read-heavy kernel?  Times a 84 MB streaming-write kernel and a 84 MB
// streaming-read kernel alone and while a D2H (or H2D) copy loop of 42 MB
// chunks runs on another stream.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a dma_interference.cu -o dma
#include <cstdio>
#include <cuda_runtime.h>

__global__ void writer(uint4* p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_uint4((unsigned)i, 1, 2, 3);
}
__global__ void sm_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}
__global__ void reader(const uint4* p, size_t n, unsigned* out) {
    unsigned acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        acc ^= __ldg(&p[i]).x;
    if (acc == 0x12345678u) *out = acc;
}

int main() {
    const size_t bytes = 84ull << 20, n = bytes / 16, cbytes = 42ull << 20;
    uint4 *dbuf, *dsrc, *ddst;
    unsigned* dout;
    void* host;
    cudaMalloc(&dbuf, bytes);
    cudaMalloc(&dsrc, cbytes);
    cudaMalloc(&ddst, cbytes);
    cudaMalloc(&dout, 4);
    cudaHostAlloc(&host, cbytes, cudaHostAllocMapped);
    void* hostd = nullptr;
    cudaHostGetDevicePointer(&hostd, host, 0);
    cudaStream_t sk, sc;
    cudaStreamCreateWithFlags(&sk, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](int kind, int dma) {
        // dma: 0 none, 1 D2H, 2 H2D, 3 both, 4 D2D (copy engine, no PCIe)
        for (int w = 0; w < 3; ++w) writer<<<148 * 8, 256, 0, sk>>>(dbuf, n);
        cudaStreamSynchronize(sk);
        if (dma & 1) for (int i = 0; i < 8; ++i) cudaMemcpyAsync(host, dsrc, cbytes, cudaMemcpyDeviceToHost, sc);
        if (dma & 2) for (int i = 0; i < 8; ++i) cudaMemcpyAsync(dsrc, host, cbytes, cudaMemcpyHostToDevice, sc);
        if (dma == 4) for (int i = 0; i < 64; ++i) cudaMemcpyAsync(ddst, dsrc, cbytes, cudaMemcpyDeviceToDevice, sc);
        if (dma == 5) for (int i = 0; i < 8; ++i) sm_copy<<<16, 256, 0, sc>>>(dsrc, (uint4*)hostd, cbytes / 16);
        if (dma == 6) for (int i = 0; i < 8; ++i) sm_copy<<<16, 256, 0, sc>>>((const uint4*)hostd, dsrc, cbytes / 16);
        float best = 1e9, tot = 0;
        for (int r = 0; r < 20; ++r) {
            cudaEventRecord(a, sk);
            if (kind == 0) writer<<<148 * 4, 256, 0, sk>>>(dbuf, n);
            else reader<<<148 * 4, 256, 0, sk>>>(dbuf, n, dout);
            cudaEventRecord(b, sk);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            tot += ms;
            if (ms < best) best = ms;
        }
        cudaDeviceSynchronize();
        printf("%-6s dma=%-5s avg %7.1f us  best %7.1f us\n", kind ? "read" : "write",
               dma == 0 ? "none" : dma == 1 ? "d2h" : dma == 2 ? "h2d" : dma == 3 ? "both" : dma == 4 ? "d2d" : dma == 5 ? "smd2h" : "smh2d", tot / 20 * 1e3,
               best * 1e3);
    };
    for (int kind = 0; kind < 2; ++kind)
        for (int dma = 0; dma < 7; ++dma) run(kind, dma);
    // host-link rate of the SM copy alone
    {
        cudaEvent_t c0, c1;
        cudaEventCreate(&c0);
        cudaEventCreate(&c1);
        for (int dir = 0; dir < 2; ++dir) {
            cudaEventRecord(c0, sc);
            for (int i = 0; i < 8; ++i)
                if (dir == 0) sm_copy<<<16, 256, 0, sc>>>(dsrc, (uint4*)hostd, cbytes / 16);
                else sm_copy<<<16, 256, 0, sc>>>((const uint4*)hostd, dsrc, cbytes / 16);
            cudaEventRecord(c1, sc);
            cudaEventSynchronize(c1);
            float ms;
            cudaEventElapsedTime(&ms, c0, c1);
            printf("sm copy %s: %.1f GB/s (16 CTAs)\n", dir ? "h2d" : "d2h", 8 * cbytes / (ms * 1e-3) / 1e9);
            cudaEventRecord(c0, sc);
            for (int i = 0; i < 8; ++i)
                cudaMemcpyAsync(dir ? (void*)dsrc : host, dir ? host : (void*)dsrc, cbytes,
                                dir ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost, sc);
            cudaEventRecord(c1, sc);
            cudaEventSynchronize(c1);
            cudaEventElapsedTime(&ms, c0, c1);
            printf("ce copy %s: %.1f GB/s\n", dir ? "h2d" : "d2h", 8 * cbytes / (ms * 1e-3) / 1e9);
        }
    }
    return 0;
}
