// common.cuh — shared host/device helpers for the EL-attention library.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>

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

}  // namespace elattn_gpu
