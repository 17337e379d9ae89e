// Programmatic dependent launch (sm_90+): a kernel launched with launch_pdl may be
// scheduled while the previous kernel on the stream is still draining; everything it
// does before pdl_wait() (shared-memory staging of read-only tables, histogram
// zeroing) overlaps that tail, and pdl_wait() blocks until the previous grid has
// completed and its writes are visible.  Every kernel launched this way calls
// pdl_wait() before it touches memory an earlier kernel wrote.
#pragma once

#include <cuda_runtime.h>

namespace etune_b200 {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace etune_b200
