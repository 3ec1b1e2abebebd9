// Programmatic dependent launch (PDL) helpers for the small-kernel chains (unfused tail,
// stochastic path): a kernel launched with launch_pdl may start while its predecessor drains,
// so every such kernel calls pdl_wait() before touching anything the predecessor writes.
// pdl_wait() / pdl_trigger() are no-ops for plain launches.  -DMCP_CFG_PDL=0 (tools/build_variant.py)
// disables the launch attribute everywhere (A/B builds).
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>

#include "tuning.h"
#include <utility>

namespace mcp {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
// the usual prologue of a chain kernel: wait for the predecessor, let the successor launch
__device__ __forceinline__ void pdl_enter() {
  pdl_wait();
  pdl_trigger();
}

inline bool pdl_enabled() { return MCP_CFG_PDL != 0; }

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace mcp
