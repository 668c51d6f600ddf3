// Programmatic dependent launch (PDL): every librdkv kernel is launched with
// programmatic stream serialization, so the next kernel's launch and prologue
// (barrier init, TMEM alloc, tensor-map prefetch) overlap the tail of the
// current one.  Each kernel calls pdl_wait() before touching global memory a
// predecessor may produce or consume; without the launch attribute the wait
// is a no-op.  Captured CUDA graphs keep the programmatic edges.
#pragma once
#include <cuda_runtime.h>

namespace rdkv {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

bool pdl_enabled();  // RDKV_PDL=0 disables (A/B measurements)

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

}  // namespace rdkv
