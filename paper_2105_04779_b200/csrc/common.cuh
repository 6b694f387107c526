// common.cuh — shared host/device helpers for the EL-attention library.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>
#include <utility>

#include "elattn_gpu.h"

namespace elattn_gpu {

// ---- element types -------------------------------------------------------
template <typename T>
__device__ __forceinline__ float to_f32(T v);
template <>
__device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T>
__device__ __forceinline__ T from_f32(float v);
template <>
__device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

inline size_t dtype_bytes(int dtype) { return dtype == ELATTN_DTYPE_BF16 ? 2 : 4; }

// ---- error plumbing ------------------------------------------------------
// Thrown inside the library only; converted to a status at the C boundary.
struct Status {
    int code;
    std::string msg;
};

void set_last_error(const std::string& msg);
void count_launch(int n = 1);

#define ELA_CHECK_CUDA(expr)                                                              \
    do {                                                                                  \
        cudaError_t _e = (expr);                                                          \
        if (_e != cudaSuccess)                                                            \
            throw ::elattn_gpu::Status{_e == cudaErrorMemoryAllocation ? ELATTN_ERR_OOM   \
                                                                       : ELATTN_ERR_CUDA, \
                                       std::string(#expr) + ": " + cudaGetErrorString(_e)}; \
    } while (0)

#define ELA_CHECK_LAUNCH()                  \
    do {                                    \
        ::elattn_gpu::count_launch();       \
        ELA_CHECK_CUDA(cudaGetLastError()); \
    } while (0)

#define ELA_REQUIRE(cond, code, msg)                            \
    do {                                                        \
        if (!(cond)) throw ::elattn_gpu::Status{(code), (msg)}; \
    } while (0)

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Programmatic dependent launch (PDL) for the kernels of a layer step: each kernel is
// launched with programmatic stream serialisation, signals launch_dependents once its
// prologue (barriers, TMEM allocation) is done and waits (griddepcontrol.wait) before
// touching data of its predecessors, so launch latency and prologue overlap the previous
// kernel's tail.  On by default; ELATTN_PDL=0 or elattn_gpu_testing_set_pdl(0) turns it off.
extern int g_pdl;  // -1 = not yet read from the environment
bool pdl_enabled();

// cudaLaunchKernelEx with optional cluster dims and the PDL attribute.
template <typename... KArgs, typename... Args>
void launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, int cluster_x,
               Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int n = 0;
    if (cluster_x > 1) {
        attr[n].id = cudaLaunchAttributeClusterDimension;
        attr[n].val.clusterDim.x = cluster_x;
        attr[n].val.clusterDim.y = 1;
        attr[n].val.clusterDim.z = 1;
        ++n;
    }
    if (pdl_enabled()) {
        attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[n].val.programmaticStreamSerializationAllowed = 1;
        ++n;
    }
    cfg.attrs = attr;
    cfg.numAttrs = n;
    ELA_CHECK_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

}  // namespace elattn_gpu
