// Programmatic dependent launch (PDL): every engine kernel is launched with
// programmatic stream serialization, calls griddepcontrol.launch_dependents
// early and griddepcontrol.wait before touching its inputs, so the next
// kernel's CTAs are scheduled and run their prologue (barrier init, TMEM
// alloc, descriptor prefetch) while this kernel drains. Inside CUDA graphs the
// edges become programmatic. TLT_PDL=0 disables it.
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <string>

#include "tlt_internal.h"

namespace tlt {

__device__ __forceinline__ void pdl_wait() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

inline bool pdl_enabled() {
    static int on = [] {
        const char* v = std::getenv("TLT_PDL");
        return v ? std::atoi(v) : 1;
    }();
    return on != 0;
}

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
    if (e != cudaSuccess) throw CudaError(std::string("launch: ") + cudaGetErrorString(e));
}

}  // namespace tlt
