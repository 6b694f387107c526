// Probe: the GEMM producer pattern — per stage an A box and a B box of 128 rows x kbp
// k-blocks (64 bf16 each, SWIZZLE_128B) from row-major [rows][K] operands viewed as 3-D
// (64, rows, K/64) tensor maps (k-block stride 128 B < row stride), consumer releases at
// once.  Measures per-SM ingress for kbp = 1, 2, 4.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                     : "=r"(ok)
                     : "r"(su32(b)), "r"(par)
                     : "memory");
}
__device__ __forceinline__ void arrive_tx(uint64_t* b, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            su32(dst)),
        "l"((uint64_t)m), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

__global__ void __launch_bounds__(32, 1)
    ingress(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, int kbp, int K, int ring,
            int reps, unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
    const int box = 128 * 128 * kbp;
    const int stage_bytes = 2 * box;
    uint64_t* full = (uint64_t*)(smem + ring * stage_bytes);
    if (threadIdx.x == 0) {
        for (int i = 0; i < ring; ++i) mbar_init(&full[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncwarp();
    if (threadIdx.x != 0) return;
    const int nk = K / 64 / kbp;
    const int iters = nk * reps;
    const int m0 = (blockIdx.x % 10) * 128, n0 = (blockIdx.x / 10 % 8) * 128;
    unsigned long long t0 = clock64();
    for (int g = 0; g < iters + ring; ++g) {
        if (g >= ring) mbar_wait(&full[g % ring], ((g / ring) - 1) & 1);
        if (g < iters) {
            const int s = g % ring, kb = (g % nk) * kbp;
            arrive_tx(&full[s], stage_bytes);
            tma3(smem + s * stage_bytes, &ta, &full[s], 0, m0, kb);
            tma3(smem + s * stage_bytes + box, &tb, &full[s], 0, n0, kb);
        }
    }
    cyc[blockIdx.x] = clock64() - t0;
}

int main() {
    cuInit(0);
    CUdevice dev;
    CUcontext ctx;
    cuDeviceGet(&dev, 0);
    cuDevicePrimaryCtxRetain(&ctx, dev);
    cuCtxSetCurrent(ctx);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    const int M = 1280, N = 1024, K = 1024;
    void *A, *B;
    cudaMalloc(&A, size_t(M) * K * 2);
    cudaMalloc(&B, size_t(N) * K * 2);
    cudaMemset(A, 1, size_t(M) * K * 2);
    cudaMemset(B, 1, size_t(N) * K * 2);
    unsigned long long* cyc;
    cudaMalloc(&cyc, 1024 * 8);
    cudaFuncSetAttribute(ingress, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    for (int kbp : {1, 2, 4}) {
        CUtensorMap ta, tb;
        cuuint64_t dA[3] = {64, (cuuint64_t)M, (cuuint64_t)K / 64}, dB[3] = {64, (cuuint64_t)N, (cuuint64_t)K / 64};
        cuuint64_t str[2] = {(cuuint64_t)K * 2, 128};
        cuuint32_t box[3] = {64, 128, (cuuint32_t)kbp};
        cuuint32_t es[3] = {1, 1, 1};
        CUresult e1 = enc(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, A, dA, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        CUresult e2 = enc(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, B, dB, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (e1 || e2) {
            printf("encode failed %d %d\n", int(e1), int(e2));
            continue;
        }
        for (int grid : {80, 148}) {
            const int stage = 2 * 128 * 128 * kbp;
            const int ring = (200 * 1024) / stage;
            const size_t smem = size_t(ring) * stage + 1024 + 64 * 8;
            for (int rep = 0; rep < 2; ++rep) {
                ingress<<<grid, 32, smem>>>(ta, tb, kbp, K, ring, 8, cyc);
                cudaDeviceSynchronize();
                std::vector<unsigned long long> h(grid);
                cudaMemcpy(h.data(), cyc, grid * 8, cudaMemcpyDeviceToHost);
                double mx = 0;
                for (auto v : h) mx = v > mx ? v : mx;
                if (rep)
                    printf("kbp %d ring %d stages grid %3d: %.1f B/cyc/SM (%s)\n", kbp, ring, grid,
                           8.0 * 2 * 128 * K * 2 / mx, cudaGetErrorString(cudaGetLastError()));
            }
        }
    }
    return 0;
}
