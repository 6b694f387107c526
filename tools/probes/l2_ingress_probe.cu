// Probe: TMA ingress bandwidth per SM from an L2-RESIDENT operand (the projection GEMMs'
// regime: weights and activations of a few MB re-read by many CTAs), as a function of
// the number of CTAs (one per SM), the box shape and the ring depth.  The consumer
// releases each stage as soon as it lands.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_ingress_probe l2_ingress_probe.cu -lcuda
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
__device__ __forceinline__ void mbar_spin(uint64_t* b, uint32_t par) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{.reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
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

// each CTA streams `iters` boxes of box_rows x 64 bf16 (SW128) from rows (cta*stride + i*box_rows) % rows
__global__ void __launch_bounds__(32, 1)
    ingress(const __grid_constant__ CUtensorMap tm, int rows, int box_rows, int box_kb, int kbs, int ring, int iters,
            int boxes_per_stage, int spin, unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
    const int stage_bytes = box_rows * 128 * box_kb * boxes_per_stage;
    uint64_t* full = (uint64_t*)(smem + ring * stage_bytes);
    if (threadIdx.x == 0) {
        for (int i = 0; i < ring; ++i) mbar_init(&full[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncwarp();
    if (threadIdx.x != 0) return;
    const int nbox_rows = rows / box_rows;
    int start = (blockIdx.x * 37) % nbox_rows;
    unsigned long long t0 = clock64();
    for (int g = 0; g < iters + ring; ++g) {
        if (g >= ring) {  // consume stage g - ring
            if (spin) mbar_spin(&full[g % ring], ((g / ring) - 1) & 1);
            else mbar_wait(&full[g % ring], ((g / ring) - 1) & 1);
        }
        if (g < iters) {
            const int s = g % ring;
            arrive_tx(&full[s], stage_bytes);
            for (int b = 0; b < boxes_per_stage; ++b) {
                const int idx = start + g * boxes_per_stage + b;
                const int r = (idx % nbox_rows) * box_rows;
                const int kb = ((idx / nbox_rows) * box_kb) % kbs;
                tma3(smem + s * stage_bytes + b * box_rows * 128 * box_kb, &tm, &full[s], 0, r, kb);
            }
        }
    }
    unsigned long long t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
}

int main() {
    CUdevice dev;
    CUcontext ctx;
    cuInit(0);
    cuDeviceGet(&dev, 0);
    cuDevicePrimaryCtxRetain(&ctx, dev);
    cuCtxSetCurrent(ctx);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    for (int big : {0, 1}) {
    const int rows = 16384, kbs = big ? 256 : 1;  // 2 MB (L2 resident) or 512 MB (DRAM)
    void* buf;
    cudaMalloc(&buf, size_t(rows) * 128 * kbs);
    cudaMemset(buf, 1, size_t(rows) * 128 * kbs);
    unsigned long long* cyc;
    cudaMalloc(&cyc, 1024 * 8);
    cudaFuncSetAttribute(ingress, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    struct Shape { int box_rows, box_kb, per_stage; };
    for (Shape sh : {Shape{32, 1, 1}, Shape{32, 1, 8}, Shape{128, 1, 1}, Shape{128, 1, 4}, Shape{128, 4, 1}}) {
        if (big) continue;
      for (int spin : {0, 1}) {
        const int box_rows = sh.box_rows;
        CUtensorMap tm;
        cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)kbs};
        cuuint64_t str[2] = {128, (cuuint64_t)rows * 128};
        cuuint32_t box[3] = {64, (cuuint32_t)box_rows, (cuuint32_t)sh.box_kb};
        cuuint32_t es[3] = {1, 1, 1};
        CUresult er = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (er != CUDA_SUCCESS) { printf("encode failed %d\n", int(er)); continue; }
        for (int ring_kb : {128}) {
            for (int grid : {148}) {
                const int stage = box_rows * 128 * sh.box_kb * sh.per_stage;
                const int ring = ring_kb * 1024 / stage;
                const int iters = (4 << 20) / stage;  // 4 MB per CTA
                const size_t smem = size_t(ring) * stage + 1024 + 64 * 8;
                for (int rep = 0; rep < 2; ++rep) {
                    cudaEvent_t e0, e1;
                    cudaEventCreate(&e0);
                    cudaEventCreate(&e1);
                    cudaEventRecord(e0);
                    ingress<<<grid, 32, smem>>>(tm, rows, box_rows, sh.box_kb, kbs, ring, iters, sh.per_stage, spin, cyc);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    std::vector<unsigned long long> h(grid);
                    cudaMemcpy(h.data(), cyc, grid * 8, cudaMemcpyDeviceToHost);
                    double mx = 0;
                    for (auto v : h) mx = v > mx ? v : mx;
                    if (rep == 1)
                        printf("spin %d %s box %3dx%d x%d/stage ring %3d KB grid %3d: %.1f B/cyc/SM, chip %.0f GB/s, %s\n",
                               spin, big ? "DRAM" : "L2  ", box_rows, sh.box_kb, sh.per_stage, ring_kb, grid,
                               double(iters) * stage / mx, double(iters) * stage * grid / (ms * 1e6),
                               cudaGetErrorString(cudaGetLastError()));
                }
            }
        }
    }
      }
    cudaFree(buf);
    }
    return 0;
}
