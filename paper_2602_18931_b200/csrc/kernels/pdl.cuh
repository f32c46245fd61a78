// Programmatic dependent launch for the forward's kernel chain: every kernel of a forward is
// launched with programmatic stream serialisation and waits (griddepcontrol.wait: the previous
// grid complete, its writes visible) right before it first reads anything the previous kernel
// produced. The next kernel's launch is processed while the previous one drains, and the GEMMs
// issue their first weight boxes (which depend on nothing) before the wait. Measured on config 3:
// 2.80 -> 2.74 s per step; an early explicit trigger was slower (2.94 s) because dependents
// parked on SMs starve the other lane's kernels. WS_PDL=0 launches fully serialised.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

#include "cuda_check.hpp"

namespace wsb {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Early trigger: only when WS_PDL_EARLY is compiled in (measured: with two concurrent lanes,
// dependents parked on SMs waiting for their primary cost more than the overlap buys); without
// it the dependents launch as the primary's CTAs exit.
#ifdef WS_PDL_EARLY
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#else
__device__ __forceinline__ void pdl_trigger() {}
#endif
// Unconditional early trigger, for grids that leave SMs idle (small-batch GEMMs): the next
// kernel's CTAs start their prologue and weight prefetch on those SMs.
__device__ __forceinline__ void pdl_trigger_now() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("WS_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// cudaLaunchKernelEx with the programmatic-serialisation attribute (and an optional cluster).
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, std::size_t smem, cudaStream_t st, int cluster_x,
                Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int n = 0;
  if (pdl_enabled()) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster_x > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = static_cast<unsigned>(cluster_x);
    at[n].val.clusterDim.y = 1;
    at[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  WS_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

}  // namespace wsb
