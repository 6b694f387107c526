// tmap.cu — TMA descriptor encoding.
#include <cudaTypedefs.h>

#include <mutex>
#include <string>

#include "common.cuh"
#include "tmap.h"

namespace elattn_gpu {

namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    static cudaError_t err = cudaSuccess;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        err = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
        if (err == cudaSuccess && q == cudaDriverEntryPointSuccess) fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    ELA_REQUIRE(fn != nullptr, ELATTN_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    return fn;
}
}  // namespace

CUtensorMap make_tmap_bf16(const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                           const uint32_t* box, int swizzle_bytes) {
    return make_tmap(base, 2, rank, dims, strides_bytes, box, swizzle_bytes);
}

CUtensorMap make_tmap(const void* base, int elem_bytes, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                      const uint32_t* box, int swizzle_bytes) {
    CUtensorMap m;
    ELA_REQUIRE(rank >= 1 && rank <= 5, ELATTN_ERR_PARAM, "tensor map rank must be 1..5");
    cuuint32_t elem_strides[5] = {1, 1, 1, 1, 1};
    cuuint64_t gdims[5], gstrides[4];
    cuuint32_t boxd[5];
    for (int i = 0; i < rank; ++i) {
        gdims[i] = dims[i];
        boxd[i] = box[i];
    }
    for (int i = 0; i + 1 < rank; ++i) gstrides[i] = strides_bytes[i];
    const CUtensorMapDataType dt = elem_bytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    CUresult r = encode_fn()(&m, dt, cuuint32_t(rank), const_cast<void*>(base),
                             gdims, gstrides, boxd, elem_strides, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                             : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                             : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    ELA_REQUIRE(r == CUDA_SUCCESS, ELATTN_ERR_UNSUPPORTED,
                "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
    return m;
}

}  // namespace elattn_gpu
