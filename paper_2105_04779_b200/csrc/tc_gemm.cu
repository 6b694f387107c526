// tc_gemm.cu — tcgen05 GEMM (placeholder until the sm_100a kernel lands).
#include "common.cuh"
#include "kernels.h"
namespace elattn_gpu {
bool tc_gemm_supported(const GemmArgs&) { return false; }
void launch_tc_gemm(const GemmArgs&, cudaStream_t) {
    throw Status{ELATTN_ERR_UNSUPPORTED, "tcgen05 GEMM not built"};
}
}  // namespace elattn_gpu
