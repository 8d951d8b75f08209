// Programmatic dependent launch (PDL): when enabled every engine kernel is
// launched with programmatic stream serialization, calls griddepcontrol.launch_dependents
// early and griddepcontrol.wait before touching its inputs, so the next
// kernel's CTAs are scheduled and run their prologue (barrier init, TMEM
// alloc, descriptor prefetch) while this kernel drains. Inside CUDA graphs the
// edges become programmatic.
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>
#include <string>
#include <unordered_set>

#include "tlt_internal.h"

namespace tlt {

__device__ __forceinline__ void pdl_wait() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}
// Kernels that allocate TMEM signal their dependents only AFTER every CTA
// holds its allocation: a PDL-launched dependent (the next GEMM) allocates
// TMEM before its own griddepcontrol.wait, so if it could start while a CTA
// of this grid had not yet allocated, that CTA's tcgen05.alloc could block on
// the dependent's columns while the dependent waits for this grid — a
// deadlock. (Dependents launch only once every CTA of this grid has issued
// launch_dependents or exited.)
__device__ __forceinline__ void pdl_wait_only() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// TLT_PDL: "gemm" = tcgen05 GEMM launches only (default), 1 = every engine
// kernel, 0 = plain stream serialization, "other" = all but the GEMMs.
// Not every kernel by default: with PDL on all of them the 7B rollout bench
// wedged in 3 of 26 runs on B200 (an SD step's first, eager, run of a new
// graph key; no mbarrier watchdog fired); 0 of 40 runs with GEMM-only PDL,
// 0 of 18 with it off, 0 of 12 with "other" (tools/gpu_hang*.sh). GEMM-only
// keeps most of the overlap (+1.6% rollout throughput over off).
inline int pdl_mask() {
    static int m = [] {
        const char* v = std::getenv("TLT_PDL");
        if (!v) return 1;
        const std::string s(v);
        if (s == "gemm") return 1;
        if (s == "other") return 2;
        return std::atoi(v) ? 3 : 0;
    }();
    return m;
}
inline bool pdl_enabled(int bit = 2) { return (pdl_mask() & bit) != 0; }

// TLT_SMEM_CARVEOUT=1: every engine kernel prefers the maximum shared-memory
// carveout, the one the tcgen05 GEMMs (226 KB) need, so the L1 / shared split
// of an SM is never reconfigured between consecutive kernels of a step (a
// reconfiguration drains the SM and keeps a PDL-launched GEMM CTA from
// co-residing with the previous kernel's tail).
inline bool smem_carveout_max() {
    static const bool on = [] {
        const char* v = std::getenv("TLT_SMEM_CARVEOUT");
        return v ? std::atoi(v) != 0 : false;
    }();
    return on;
}

template <typename... KArgs>
inline void set_max_carveout(void (*kern)(KArgs...)) {
    if (!smem_carveout_max()) return;
    static std::mutex mu;
    static std::unordered_set<const void*> done;
    std::lock_guard<std::mutex> lk(mu);
    if (done.insert(reinterpret_cast<const void*>(kern)).second)
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
}

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
    set_max_carveout(kern);
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
