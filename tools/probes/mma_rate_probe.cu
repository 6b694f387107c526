// Probe: cycles per tcgen05.mma (kind::f16, cta_group::1) for the decode kernel's
// shapes, issued back to back by one thread, operands in smem (SS) or A in TMEM (TS).
// Also: two issuer warps concurrently.  Reports clock64 cycles / MMA at completion.
#include <cstdint>
#include <cstdio>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo) {
    uint64_t d = 0;
    d |= (addr >> 4) & 0x3FFF;
    d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
    d |= uint64_t(1024 >> 4) << 32;
    d |= 1ull << 46;
    d |= 2ull << 61;
    return d;
}
__device__ __forceinline__ uint32_t idesc(uint32_t M, uint32_t N, uint32_t amn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (amn << 15) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
template <int MODE>  // 0: SS M64N32, 1: TS M64N32, 2: SS M128N64 (A MN-major), 3: SS M64N64, 4: TS M64N64, 5: SS M128N128
__global__ void probe(int iters, int issuers, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t slot;
    __shared__ uint64_t bar[2];
    int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3c003c00u;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[1])));
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t tm = slot;
    long long t0 = clock64();
    if (warp < issuers && lane == 0) {
        uint32_t base = su32(smem) + warp * 32768;
        uint32_t d = tm + warp * 128;
        for (int i = 0; i < iters; ++i) {
            uint32_t acc = i > 0;
            if (MODE == 0 || MODE == 3) {
                const uint32_t id = idesc(64, MODE == 0 ? 32 : 64, 0);
                asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(d),
                             "l"(sdesc(base, 0)), "l"(sdesc(base + 16384, 0)), "r"(id), "r"(acc));
            } else if (MODE == 1 || MODE == 4) {
                const uint32_t id = idesc(64, MODE == 1 ? 32 : 64, 0);
                asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}" ::"r"(d),
                             "r"(tm + 256 + warp * 64), "l"(sdesc(base + 16384, 0)), "r"(id), "r"(acc));
            } else if (MODE == 2) {
                const uint32_t id = idesc(128, 64, 1);
                asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(d),
                             "l"(sdesc(base, 4096)), "l"(sdesc(base + 16384, 0)), "r"(id), "r"(acc));
            } else {
                const uint32_t id = idesc(128, 128, 0);
                asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(d),
                             "l"(sdesc(base, 0)), "l"(sdesc(base + 16384, 0)), "r"(id), "r"(acc));
            }
        }
        long long t_issued = clock64();
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[warp]))
                     : "memory");
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                         : "=r"(ok)
                         : "r"(su32(&bar[warp])));
        long long t1 = clock64();
        out[warp * 2] = t_issued - t0;
        out[warp * 2 + 1] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}
int main() {
    long long* d;
    cudaMalloc(&d, 64);
    const char* names[] = {"SS M64 N32", "TS M64 N32", "SS M128 N64 (A MN)", "SS M64 N64", "TS M64 N64", "SS M128 N128"};
    for (int mode = 0; mode < 6; ++mode)
        for (int issuers : {1, 2}) {
            const int iters = 512;
            long long h[4] = {0, 0, 0, 0};
            auto run = [&](auto kern) {
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
                kern<<<1, 64, 65536>>>(iters, issuers, d);
            };
            if (mode == 0) run(probe<0>);
            if (mode == 1) run(probe<1>);
            if (mode == 2) run(probe<2>);
            if (mode == 3) run(probe<3>);
            if (mode == 4) run(probe<4>);
            if (mode == 5) run(probe<5>);
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
            printf("%-20s issuers=%d: issue %.1f cyc/mma, complete %.1f cyc/mma (%s)\n", names[mode], issuers,
                   double(h[0]) / iters, double(h[1]) / iters, cudaGetErrorString(e));
        }
}
