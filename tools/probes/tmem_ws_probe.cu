// Probe: tcgen05.mma.ws (weight-stationary) kind::f16, M=64 N=64 K=16, A from TMEM or smem,
// D at TMEM lane offset 0 / 32 / 64.  Question: can an M=64 .ws accumulator (or A operand)
// live in the upper TMEM lanes, so that a score accumulator and the q' A operand share
// columns?  Prints the error vs fp64 and where the rows landed.
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
constexpr int M = 64, N = 64, K = 64;
// mode 0: A smem, D lane off = doff; mode 1: A tmem at lane aoff, D lane off = doff
__global__ void probe(const float* A, const float* Bm, float* D, int mode, int aoff, int doff) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t slot;
    __shared__ uint64_t bar;
    int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    uint8_t* sa = smem;          // A: 64 rows x 128 B (K=64 bf16), SW128 K-major
    uint8_t* sb = smem + 8192;   // B: 64 rows x 128 B
    for (int idx = threadIdx.x; idx < 64 * K; idx += blockDim.x) {
        int r = idx / K, k = idx % K;
        int c = k / 8, w = k % 8;
        ((__nv_bfloat16*)(sa + r * 128))[((c ^ (r & 7)) * 8) + w] = __float2bfloat16(A[r * K + k]);
        ((__nv_bfloat16*)(sb + r * 128))[((c ^ (r & 7)) * 8) + w] = __float2bfloat16(Bm[r * K + k]);
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t tm = slot;
    // zero the D region (all lanes, columns 0..63)
    {
        uint32_t z[16];
        for (int i = 0; i < 16; ++i) z[i] = 0;
        for (int c = 0; c < 64; c += 16)
            asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
                             tm + ((warp * 32) << 16) + c),
                         "r"(z[0]), "r"(z[1]), "r"(z[2]), "r"(z[3]), "r"(z[4]), "r"(z[5]), "r"(z[6]), "r"(z[7]), "r"(z[8]),
                         "r"(z[9]), "r"(z[10]), "r"(z[11]), "r"(z[12]), "r"(z[13]), "r"(z[14]), "r"(z[15]));
    }
    if (mode == 1) {
        // A into TMEM columns 128.. : row i of A in lane aoff + i (hypothesis for .ws M=64: rows in
        // consecutive lanes), bf16 pairs packed per column
        for (int half = 0; half < K / 32; ++half) {
            uint32_t v[16];
            for (int c = 0; c < 16; ++c) {
                int lanei = warp * 32 + lane, row = lanei - aoff;
                bool mine = row >= 0 && row < 64;
                float a0 = mine ? A[row * K + half * 32 + 2 * c] : 0.f, a1 = mine ? A[row * K + half * 32 + 2 * c + 1] : 0.f;
                __nv_bfloat162 h = __floats2bfloat162_rn(a0, a1);
                v[c] = *(uint32_t*)&h;
            }
            asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
                             tm + ((warp * 32) << 16) + 128 + half * 16),
                         "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
                         "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
        }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (threadIdx.x == 0) {
        uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
        uint32_t d_addr = tm + (uint32_t(doff) << 16);
        for (int s = 0; s < K / 16; ++s) {
            uint64_t b = sdesc(su32(sb) + 32 * s);
            uint32_t acc = s > 0;
            if (mode == 0) {
                uint64_t a = sdesc(su32(sa) + 32 * s);
                asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.ws.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(d_addr),
                             "l"(a), "l"(b), "r"(idesc), "r"(acc));
            } else {
                uint32_t a_addr = tm + (uint32_t(aoff) << 16) + 128 + 8 * s;
                asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.ws.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}" ::"r"(d_addr),
                             "r"(a_addr), "l"(b), "r"(idesc), "r"(acc));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    }
    {
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(su32(&bar)));
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int c0 = 0; c0 < 64; c0 += 32) {
        uint32_t r[32];
        uint32_t t = tm + ((warp * 32) << 16) + c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%"
            "21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
              "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
              "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
              "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(t));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int c = 0; c < 32; ++c) D[(warp * 32 + lane) * 64 + c0 + c] = __uint_as_float(r[c]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}
int main() {
    static float hA[M * K], hB[N * K], hD[128 * 64], ref[M * N];
    for (int i = 0; i < M * K; ++i) hA[i] = float((i * 37) % 17 - 8) / 8.f;
    for (int i = 0; i < N * K; ++i) hB[i] = float((i * 53) % 13 - 6) / 4.f;
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < N; ++j) {
            double s = 0;
            for (int k = 0; k < K; ++k)
                s += double(__bfloat162float(__float2bfloat16(hA[i * K + k]))) * __bfloat162float(__float2bfloat16(hB[j * K + k]));
            ref[i * N + j] = float(s);
        }
    float *A, *Bm, *D;
    cudaMalloc(&A, sizeof hA);
    cudaMalloc(&Bm, sizeof hB);
    cudaMalloc(&D, sizeof hD);
    cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice);
    cudaMemcpy(Bm, hB, sizeof hB, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    struct C { int mode, aoff, doff; } cs[] = {{0, 0, 0}, {0, 0, 64}, {0, 0, 32}, {1, 0, 0}, {1, 0, 64}, {1, 64, 0}};
    for (auto c : cs) {
        cudaMemset(D, 0, sizeof hD);
        probe<<<1, 128, 32768>>>(A, Bm, D, c.mode, c.aoff, c.doff);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
        // locate each reference row among the 128 lanes
        int found = 0, first_lane = -1, last_lane = -1;
        double maxerr = 0;
        for (int i = 0; i < M; ++i) {
            int hit = -1;
            for (int l = 0; l < 128 && hit < 0; ++l) {
                bool ok = true;
                for (int j = 0; j < N && ok; ++j) ok = fabs(hD[l * 64 + j] - ref[i * N + j]) < 1e-2;
                if (ok) hit = l;
            }
            if (hit >= 0) {
                ++found;
                if (i == 0) first_lane = hit;
                if (i == M - 1) last_lane = hit;
            }
        }
        printf("mode=%s aoff=%d doff=%d err=%s rows_found=%d row0->lane %d row63->lane %d\n", c.mode ? "A_tmem" : "A_smem",
               c.aoff, c.doff, cudaGetErrorString(e), found, first_lane, last_lane);
        if (e != cudaSuccess) break;
    }
}
