// Probe: achievable HBM bandwidth for the decode kernel's H access pattern with
// TMA (per input, d_m split across a CTA pair, tiles of `rows` x 128 columns
// per unit), as a function of ring depth.  The consumer releases each unit as
// soon as it lands, so this is the memory system's ceiling for the pattern.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
    uint32_t ok = 0;
    while (!ok) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(su32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void arrive_tx(uint64_t* b, uint32_t tx) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(tx) : "memory"); }
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                 ::"r"(su32(dst)), "l"((uint64_t)m), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}

template <int ROWS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(64, 1)
stream(const __grid_constant__ CUtensorMap tm, int n, int d_m, int ring, int B) {
    extern __shared__ __align__(1024) uint8_t smem[];
    constexpr int kUnit = ROWS * 128 * 2;
    uint64_t* full = (uint64_t*)(smem + ring * kUnit);
    uint64_t* empty = full + ring;
    int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    uint32_t rank; asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    if (threadIdx.x == 0) { for (int i = 0; i < ring; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); } asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncthreads();
    const int units_per_tile = d_m / 2 / 128;
    const int tiles = n / ROWS;
    for (int b = blockIdx.x / 2; b < B; b += gridDim.x / 2) {
      const int total = tiles * units_per_tile;
      if (warp == 0 && lane == 0) {
        for (int g = 0; g < total; ++g) {
            static __shared__ int gg; (void)gg;
            const int s = g % ring;
            const int use = g / ring;
            mbar_wait(&empty[s], (use & 1) ^ 1);
            arrive_tx(&full[s], kUnit);
            const int j = g / units_per_tile, u = g % units_per_tile;
            const int col = rank * (d_m / 2) + 128 * u;
            tma3(smem + s * kUnit, &tm, &full[s], col, j * ROWS, b);
            tma3(smem + s * kUnit + kUnit / 2, &tm, &full[s], col + 64, j * ROWS, b);
        }
      } else if (warp == 1 && lane == 0) {
        for (int g = 0; g < total; ++g) {
            const int s = g % ring;
            mbar_wait(&full[s], (g / ring) & 1);
            arrive(&empty[s]);
        }
      }
      __syncthreads();
      // reset barrier parity bookkeeping per input: re-init (all idle now)
      if (threadIdx.x == 0) { for (int i = 0; i < ring; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); } asm volatile("fence.mbarrier_init.release.cluster;"); }
      __syncthreads();
    }
}

int main() {
    const int B = 320, n = 1024, d_m = 1024;
    size_t bytes = (size_t)B * n * d_m * 2;
    void* H; cudaMalloc(&H, bytes); cudaMemset(H, 0, bytes);
    PFN_cuTensorMapEncodeTiled_v12000 enc; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    for (int rows : {32, 64}) {
      CUtensorMap tm;
      cuuint64_t dims[3] = {(cuuint64_t)d_m, (cuuint64_t)n, (cuuint64_t)B};
      cuuint64_t str[2] = {(cuuint64_t)d_m * 2, (cuuint64_t)n * d_m * 2};
      cuuint32_t box[3] = {64, (cuuint32_t)rows, 1}, es[3] = {1, 1, 1};
      enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, H, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      for (int ring_kb : {32, 64, 96, 128, 160, 192}) {
        int unit = rows * 256;
        int ring = ring_kb * 1024 / unit;
        size_t smem = ring * unit + 2 * ring * 8 + 64;
        for (int persistent : {0, 1}) {
          int grid = persistent ? 148 : 2 * B;
          if (rows == 32) cudaFuncSetAttribute(stream<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
          else cudaFuncSetAttribute(stream<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
          cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
          for (int it = 0; it < 3; ++it) { if (rows == 32) stream<32><<<grid, 64, smem>>>(tm, n, d_m, ring, B); else stream<64><<<grid, 64, smem>>>(tm, n, d_m, ring, B); }
          cudaEventRecord(e0);
          const int reps = 5;
          for (int it = 0; it < reps; ++it) { if (rows == 32) stream<32><<<grid, 64, smem>>>(tm, n, d_m, ring, B); else stream<64><<<grid, 64, smem>>>(tm, n, d_m, ring, B); }
          cudaEventRecord(e1); cudaEventSynchronize(e1);
          float ms; cudaEventElapsedTime(&ms, e0, e1);
          cudaError_t err = cudaGetLastError();
          printf("rows=%d ring=%3d KB persistent=%d : %.1f us  %.0f GB/s  %s\n", rows, ring_kb, persistent, ms / reps * 1e3,
                 bytes / (ms / reps * 1e-3) / 1e9, cudaGetErrorString(err));
        }
      }
    }
}
