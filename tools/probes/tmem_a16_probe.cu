// Probe: tcgen05.mma kind::f16 with the M=64 A operand in TMEM at lane offset 0 or 16
// (rows in lanes 16..31 of each quadrant: would let two M=64 A operands share columns),
// D at lane offset 0, B K-major SW128 in smem.
// Hypothesis: A row i lives in TMEM lane (i%16) + 32*(i/16); K element k of a
// row is bf16 #(k%2) of 32-bit column (k/2); K-step s reads columns [8s, 8s+8).
#include <cuda_bf16.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
    uint64_t d = 0;
    d |= (addr >> 4) & 0x3FFF;
    d |= uint64_t(1024 >> 4) << 32;
    d |= 1ull << 46;
    d |= 2ull << 61;
    return d;
}
constexpr int M = 64, N = 32, K = 64;
__global__ void probe(const float* A, const float* Bm, float* D, int a_off) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t slot;
    __shared__ uint64_t bar;
    int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (int idx = threadIdx.x; idx < N * K; idx += blockDim.x) {
        int r = idx / K, k = idx % K;
        __nv_bfloat16* row = (__nv_bfloat16*)(smem + r * 128);
        int c = k / 8, w = k % 8;
        row[((c ^ (r & 7)) * 8) + w] = __float2bfloat16(Bm[r * K + k]);
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t tm = slot;
    for (int half = 0; half < K / 32; ++half) {
        uint32_t v[16];
        for (int c = 0; c < 16; ++c) {
            const bool mine = a_off ? lane >= 16 : lane < 16;
            int row = 16 * warp + (lane & 15);
            float a0 = mine ? A[row * K + half * 32 + 2 * c] : 7.f;
            float a1 = mine ? A[row * K + half * 32 + 2 * c + 1] : 7.f;
            __nv_bfloat162 h = __floats2bfloat162_rn(a0, a1);
            v[c] = *(uint32_t*)&h;
        }
        uint32_t t = tm + ((warp * 32) << 16) + 64 + half * 16;
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(t),
            "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
            "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (threadIdx.x == 0) {
        uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
        uint32_t d_addr = tm;
        for (int s = 0; s < K / 16; ++s) {
            uint32_t a_addr = tm + (uint32_t(a_off) << 16) + 64 + 8 * s;
            uint64_t b = sdesc(su32(smem) + 32 * s);
            uint32_t acc = s > 0;
            asm volatile(
                "{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}" ::"r"(d_addr),
                "r"(a_addr), "l"(b), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                     : "memory");
    }
    {
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                         : "=r"(ok)
                         : "r"(su32(&bar)));
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t r[32];
    uint32_t t = tm + ((warp * 32) << 16);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%"
        "21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(t));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int c = 0; c < 32; ++c) D[(warp * 32 + lane) * 32 + c] = __uint_as_float(r[c]);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm));
}
int main() {
    static float hA[M * K], hB[N * K], hD[128 * 32];
    for (int i = 0; i < M * K; ++i) hA[i] = float((i * 37) % 17 - 8) / 8.f;
    for (int i = 0; i < N * K; ++i) hB[i] = float((i * 53) % 13 - 6) / 4.f;
    float *A, *Bm, *D;
    cudaMalloc(&A, sizeof hA);
    cudaMalloc(&Bm, sizeof hB);
    cudaMalloc(&D, sizeof hD);
    cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice);
    cudaMemcpy(Bm, hB, sizeof hB, cudaMemcpyHostToDevice);
    for (int lane_off : {0, 16}) {
        cudaMemset(D, 0, sizeof hD);
        probe<<<1, 128, 8192>>>(A, Bm, D, lane_off);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
        double maxerr = 0;
        int bad = 0;
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < N; ++j) {
                double ref = 0;
                for (int k = 0; k < K; ++k)
                    ref += double(__bfloat162float(__float2bfloat16(hA[i * K + k]))) *
                           __bfloat162float(__float2bfloat16(hB[j * K + k]));
                int lanei = (i % 16) + 32 * (i / 16);
                double got = hD[lanei * 32 + j];
                maxerr = fmax(maxerr, fabs(got - ref));
                if (fabs(got - ref) > 1e-2) ++bad;
            }
        printf("a_lane_off=%d err=%s maxerr=%.4g bad=%d\n", lane_off, cudaGetErrorString(e), maxerr, bad);
    }
}
