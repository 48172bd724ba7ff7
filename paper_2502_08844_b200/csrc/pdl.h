// pdl.h -- programmatic dependent launch for the small kernels of the PPO step
// chain: the next kernel's launch (grid placement, CTA start) overlaps the
// previous kernel's tail; the kernel waits (griddepcontrol.wait) before its
// first access to anything the previous kernel may touch.  In a kernel launched
// without the attribute the wait returns at once.
#pragma once
#include <cuda_runtime.h>

#include <utility>

namespace dk {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace dk
