// tmap.h — host-side TMA tensor-map encoding (cuTensorMapEncodeTiled via the
// runtime's driver entry point, so the library needs no -lcuda).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace elattn_gpu {

// bf16 tensor map with up to 5 dims (dim 0 innermost, contiguous; the other strides need
// not be monotonic, e.g. a k-block dimension of stride 128 B inside [rows][K]).
// dims/box in elements, strides (for dims 1..rank-1) in bytes; swizzle_bytes in
// {0, 32, 64, 128} (default SWIZZLE_128B); out-of-bounds elements are filled with zeros
// on loads and clipped on stores.
CUtensorMap make_tmap_bf16(const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                           const uint32_t* box, int swizzle_bytes = 128);
// same for bf16 (elem_bytes 2) or fp32 (elem_bytes 4) elements
CUtensorMap make_tmap(const void* base, int elem_bytes, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                      const uint32_t* box, int swizzle_bytes = 128);

}  // namespace elattn_gpu
