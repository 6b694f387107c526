// el_decode_tc.cu — tcgen05 fused EL decode (placeholder until the sm_100a kernel lands).
#include "common.cuh"
#include "kernels.h"
namespace elattn_gpu {
bool el_decode_tc_supported(int, int) { return false; }
void launch_el_decode_tc(const void*, const void*, const int*, int, int, int, int, float, void*,
                         cudaStream_t) {
    throw Status{ELATTN_ERR_UNSUPPORTED, "tcgen05 decode not built"};
}
}  // namespace elattn_gpu
