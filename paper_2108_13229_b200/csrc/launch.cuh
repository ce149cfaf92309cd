// Kernel launch with programmatic dependent launch (PDL).
//
// Every kernel of the library begins with pdl_begin(): griddepcontrol.wait
// (the previous kernel in the stream has completed and its memory is
// visible) and griddepcontrol.launch_dependents (the next kernel may be
// launched now).  Launches carry the programmatic-stream-serialization
// attribute, so the launch latency and the prologue of kernel k+1 overlap the
// tail of kernel k, also inside the captured BiCGSTAB graph.  The Gauss-Seidel
// walk does its shared-memory setup before its producer waits (gs_walk.cu).
// SDG_PDL=0 launches plainly (the kernels' waits are then no-ops).
#pragma once

#include <string>

#include "common.hpp"

namespace sdg {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_begin() {
    pdl_wait();
    pdl_trigger();
}

template <typename... KArgs, typename... Args>
inline void launch_k(Context& c, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = c.pdl ? 1 : 0;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
    if (e != cudaSuccess) fail(SDG_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
}

}  // namespace sdg
