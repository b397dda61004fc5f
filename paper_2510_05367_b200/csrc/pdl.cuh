// Programmatic dependent launch (PDL).  Kernels on the compute stream are
// launched with cudaLaunchAttributeProgrammaticStreamSerialization, so a
// kernel's CTAs can be scheduled on SMs freed by the previous kernel's tail
// and run their prologue (barrier init, TMEM allocation, descriptor
// prefetch) while it drains.  Every such kernel calls pdl_wait() before its
// first access to data another kernel writes or reads: griddepcontrol.wait
// returns once the preceding grid has completed and its writes are visible
// (a no-op for a kernel launched without the attribute).  LC_PDL=0 turns the
// attribute off.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

namespace lc {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Let the next kernel's grid be scheduled now (persistent kernels whose CTAs
// are all resident: its CTAs take SMs as this grid's CTAs exit).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline bool pdl_enabled() {
    static const bool on = !(std::getenv("LC_PDL") && std::atoi(std::getenv("LC_PDL")) == 0);
    return on;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace lc
