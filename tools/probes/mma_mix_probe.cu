// Probe: the decode kernel's tcgen05.mma MIX on one SM — two score issuers plus one O
// issuer running concurrently, as in el_decode_tc.cu — to measure tensor-pipe time per
// 32-row tile for score MMAs of N = 32 (one tile per MMA chain) vs N = 64 (two tiles).
//   score MMAs: M64, K16, half with A from TMEM (TS), half with A from smem (SS)
//   O MMAs:     M128 N64 K16, A MN-major from smem (LBO 4 KB), 8 per tile
// Reports cycles per tile from first issue to the last commit's completion.
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
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(d),
                 "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}" ::"r"(d),
                 "r"(a), "l"(b), "r"(id), "r"(acc));
}
// tiles: 32-row tiles to score; n_sc: score N (32 or 64); s_issuers: 0..2; o_on: O issuer active
__global__ void probe(int tiles, int n_sc, int s_issuers, int o_on, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t slot;
    __shared__ uint64_t bar[3];
    int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (int i = threadIdx.x; i < 196608 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3c003c00u;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0)
        for (int i = 0; i < 3; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = slot;
    const uint32_t q = su32(smem), ringb = q + 32768;  // q' smem half (32 KB), ring (160 KB)
    long long t0 = clock64();
    bool active = (warp < 2 && warp < s_issuers) || (warp == 2 && o_on);
    if (active && lane == 0) {
        if (warp < 2) {
            const uint32_t id = idesc(64, n_sc, 0);
            const int groups = tiles / (n_sc / 32);
            const uint32_t d = tm + warp * 64;
            for (int gi = warp; gi < groups; gi += s_issuers) {
                const uint32_t tb = ringb + (gi % 4) * 32768;
                for (int u = 0; u < 4; ++u)
                    for (int kk = 0; kk < 8; ++kk) {
                        const uint64_t bd = sdesc(tb + u * 8192 + (kk >> 2) * 4096 + 32 * (kk & 3), 0);
                        const uint32_t acc = (u | kk) != 0;
                        if (u < 2)
                            mma_ts(d, tm + 384 + u * 64 + kk * 8, bd, id, acc);
                        else
                            mma_ss(d, sdesc(q + ((2 * (u - 2) + (kk >> 2)) * 8192 + 32 * (kk & 3)), 0), bd, id, acc);
                    }
            }
        } else {
            const uint32_t id = idesc(128, 64, 1);
            for (int t = 0; t < tiles; ++t) {
                const uint32_t tb = ringb + (t % 4) * 32768;
                for (int m = 0; m < 4; ++m)
                    for (int kk = 0; kk < 2; ++kk)
                        mma_ss(tm + 128 + m * 64, sdesc(tb + m * 8192 + kk * 2048, 4096),
                               sdesc(q + 16384 + 32 * kk, 0), id, (t | kk) != 0);
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[warp]))
                     : "memory");
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                         : "=r"(ok)
                         : "r"(su32(&bar[warp])));
        out[warp] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}
int main() {
    long long* d;
    cudaMalloc(&d, 64);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608);
    const int tiles = 256;
    struct Cfg { int n, s, o; const char* name; } cfgs[] = {
        {32, 2, 0, "S N32 x2 issuers, no O"}, {64, 2, 0, "S N64 x2 issuers, no O"},
        {32, 1, 0, "S N32 x1 issuer, no O"},  {64, 1, 0, "S N64 x1 issuer, no O"},
        {32, 0, 1, "O only"},                 {32, 2, 1, "S N32 x2 + O (old decode mix)"},
        {64, 2, 1, "S N64 x2 + O (paired mix)"}, {64, 1, 1, "S N64 x1 + O"}};
    for (auto& c : cfgs) {
        long long h[3] = {0, 0, 0};
        cudaMemset(d, 0, 64);
        probe<<<1, 96, 196608>>>(tiles, c.n, c.s, c.o, d);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
        long long mx = h[0] > h[1] ? h[0] : h[1];
        mx = mx > h[2] ? mx : h[2];
        printf("%-34s cycles/tile %.1f  (S0 %.1f, S1 %.1f, O %.1f) %s\n", c.name, double(mx) / tiles, double(h[0]) / tiles,
               double(h[1]) / tiles, double(h[2]) / tiles, cudaGetErrorString(e));
    }
}
