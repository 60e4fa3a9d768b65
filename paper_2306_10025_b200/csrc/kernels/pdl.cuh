// Programmatic dependent launch (sm_90+), shared by the sweep kernels.
//
// The sweep's kernels are launched with programmatic stream serialization:
// each one issues the loads that do not depend on its predecessor (matrix
// values/columns, tile indices, inverse-map slots, x) before
// griddepcontrol.wait, which returns once the predecessor grid has completed
// and its writes are visible.  Each kernel lets its dependent launch only
// after its own wait (so completion stays transitive along the stream); the
// dependent's CTAs then occupy SMs freed by the primary's last wave.
// Without the launch attribute both instructions are no-ops.  PDB_PDL=0
// launches without the attribute (A/B).
#pragma once

#include <cstdlib>

#include <cuda_runtime.h>

namespace pdb::k {

__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline bool pdl_enabled() {
  const char* e = getenv("PDB_PDL");
  return !(e && e[0] == '0');
}

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

}  // namespace pdb::k
