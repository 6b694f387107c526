// mha.cu — the multi-head-attention baseline path on the GPU (the reference's MHA with a
// per-head K/V cache: multi_head_attention, attention.hpp:96-113; KvCache::append /
// attention_over_cache, :118-180), built from this library's own kernels so EL and MHA
// are compared on the same B200 with the same GEMMs:
//   (1) K_i = H.W_K,i (+ b_K,i), V_i = H.W_V,i (+ b_V,i) for every input: two head-batched
//       GEMMs (tc_gemm on bf16, SIMT on fp32) into caches [h][B][n][d_k];
//   (2) Q = Y.W_Q + b_Q (GEMM);
//   (3) mha_decode_kernel: per (input b, head i) one CTA streams K_i(b) and V_i(b) once for
//       all x beam rows of the input — scores, online softmax (exp2, running max / sum),
//       P.V — into ctx [B*x][h*d_k] (fp32 accumulate);
//   (4) out = ctx.W_O + b_O (GEMM).
// Per decoder step the cache read is 2 * n * h * d_k values per input: twice the EL
// decode's single pass over H at d_m = h * d_k — the saving EL-attention is about.
#include "common.cuh"
#include "kernels.h"

namespace elattn_gpu {

namespace {

constexpr int kMhaTile = 64;      // keys per tile
constexpr int kMhaThreads = 128;  // 4 warps; warp w owns beam rows w, w + 4, ...
constexpr int kMhaMaxDk = 128;

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, bool valid) {
    // 16-byte async copy global -> shared (zero-filled when !valid)
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
    const int n = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(gsrc), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// 8 consecutive elements of a row in shared memory (16 B of bf16 / 32 B of fp32) as floats
__device__ __forceinline__ void lds8(const __nv_bfloat16* p, float (&f)[8]) {
    const uint4 v = *reinterpret_cast<const uint4*>(p);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 t = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
        f[2 * i] = t.x, f[2 * i + 1] = t.y;
    }
}
__device__ __forceinline__ void lds8(const float* p, float (&f)[8]) {
    const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
    f[0] = a.x, f[1] = a.y, f[2] = a.z, f[3] = a.w, f[4] = b.x, f[5] = b.y, f[6] = b.z, f[7] = b.w;
}
__device__ __forceinline__ float2 lds2(const __nv_bfloat16* p) {
    return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(p));
}
__device__ __forceinline__ float2 lds2(const float* p) { return *reinterpret_cast<const float2*>(p); }

// ctx[(b*x + r)][i*d_k + c] = softmax_t(Q_r,i . K_i(b)[t] * scale) . V_i(b)[t][c]
// Q [B*x][h*d_k], K/V [h][B][n_stride][d_k], all of type T; npi (optional) context lengths.
// K/V tiles of 64 keys stream through a cp.async double buffer in their storage type (rows
// padded by 16 bytes: the 8 lanes of a 16-byte load wavefront reading 8 keys hit 8
// different bank quads); scores and P.V accumulate in fp32.
template <typename T>
__global__ void __launch_bounds__(kMhaThreads)
    mha_decode_kernel(const T* __restrict__ Q, const T* __restrict__ Kc, const T* __restrict__ Vc,
                      const int* __restrict__ npi, int B, int x, int h, int d_k, int n_stride, float scale_log2,
                      T* __restrict__ ctx) {
    extern __shared__ __align__(16) uint8_t sm_raw[];
    constexpr int kE = 16 / int(sizeof(T));  // elements per 16 bytes
    const int ld = d_k + kE;                 // padded row (elements)
    T* sKV = reinterpret_cast<T*>(sm_raw);   // [2 stages][K, V][kMhaTile][ld]
    float* sQ = reinterpret_cast<float*>(sm_raw + size_t(2) * 2 * kMhaTile * ld * sizeof(T));  // [x][d_k]
    float* sP = sQ + x * d_k;                                                                     // [4][kMhaTile]
    const int b = blockIdx.x, i = blockIdx.y, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int n_b = npi ? npi[b] : n_stride;
    const int hk = h * d_k;
    if (n_b < 1 || n_b > n_stride) {  // out-of-contract context length: loud NaN rows
        for (int e = tid; e < x * d_k; e += kMhaThreads)
            ctx[int64_t(b * x + e / d_k) * hk + i * d_k + e % d_k] = from_f32<T>(__int_as_float(0x7fc00000));
        return;
    }
    for (int e = tid; e < x * d_k; e += kMhaThreads)
        sQ[e] = to_f32<T>(Q[int64_t(b * x + e / d_k) * hk + i * d_k + e % d_k]);
    const int64_t base = (int64_t(i) * B + b) * n_stride * d_k;
    const T* Kb = Kc + base;
    const T* Vb = Vc + base;
    const int chunks = d_k / kE;  // 16-byte chunks per row
    auto load_tile = [&](int tt) {
        T* st = sKV + size_t(tt & 1) * 2 * kMhaTile * ld;
        for (int v = tid; v < 2 * kMhaTile * chunks; v += kMhaThreads) {
            const int which = v / (kMhaTile * chunks), e = v % (kMhaTile * chunks);
            const int key = e / chunks, c = (e % chunks) * kE, t = tt * kMhaTile + key;
            const bool ok = t < n_b;
            cp_async16(st + (which * kMhaTile + key) * ld + c, (which ? Vb : Kb) + int64_t(ok ? t : 0) * d_k + c, ok);
        }
        cp_async_commit();
    };
    constexpr int kRowsPerWarp = 4;  // x <= 16
    constexpr int kPairs = kMhaMaxDk / 64;
    float m[kRowsPerWarp], l[kRowsPerWarp], acc[kRowsPerWarp][2 * kPairs];
#pragma unroll
    for (int r = 0; r < kRowsPerWarp; ++r) {
        m[r] = -INFINITY, l[r] = 0.f;
#pragma unroll
        for (int j = 0; j < 2 * kPairs; ++j) acc[r][j] = 0.f;
    }
    const int T_all = (n_b + kMhaTile - 1) / kMhaTile;
    load_tile(0);
    for (int tt = 0; tt < T_all; ++tt) {
        cp_async_wait_all();
        __syncthreads();  // tile tt landed for every thread; tile tt - 1's buffer is free
        if (tt + 1 < T_all) load_tile(tt + 1);
        const T* sK = sKV + size_t(tt & 1) * 2 * kMhaTile * ld;
        const T* sV = sK + kMhaTile * ld;
        const int nvalid = min(kMhaTile, n_b - tt * kMhaTile);
#pragma unroll
        for (int rr = 0; rr < kRowsPerWarp; ++rr) {
            const int r = warp + 4 * rr;
            if (r >= x) break;
            // scores of keys lane and lane + 32
            float s0 = 0.f, s1 = 0.f;
            const float* q = sQ + r * d_k;
            for (int c = 0; c < d_k; c += 8) {
                float a[8], bb[8];
                lds8(sK + lane * ld + c, a);
                lds8(sK + (lane + 32) * ld + c, bb);
                const float4 q0 = *reinterpret_cast<const float4*>(q + c), q1 = *reinterpret_cast<const float4*>(q + c + 4);
                const float qv[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
#pragma unroll
                for (int u = 0; u < 8; ++u) s0 = fmaf(qv[u], a[u], s0), s1 = fmaf(qv[u], bb[u], s1);
            }
            if (lane >= nvalid) s0 = -INFINITY;
            if (lane + 32 >= nvalid) s1 = -INFINITY;
            float tmax = fmaxf(s0, s1);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
            const float m_new = fmaxf(m[rr], tmax);
            const float alpha = exp2f((m[rr] - m_new) * scale_log2);  // 0 on the first tile
            const float p0 = exp2f((s0 - m_new) * scale_log2), p1 = exp2f((s1 - m_new) * scale_log2);
            float psum = p0 + p1;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) psum += __shfl_xor_sync(0xffffffffu, psum, o);
            l[rr] = l[rr] * alpha + psum;
            m[rr] = m_new;
            float* p = sP + warp * kMhaTile;
            p[lane] = p0;
            p[lane + 32] = p1;
            __syncwarp();
            // P.V: lane owns column pairs c = 2 lane + 64 j; keys past nvalid have p = 0 and
            // zero-filled V rows
#pragma unroll
            for (int j = 0; j < kPairs; ++j) {
                const int c = 2 * lane + 64 * j;
                if (c < d_k) {
                    float a0 = acc[rr][2 * j] * alpha, a1 = acc[rr][2 * j + 1] * alpha;
                    for (int k = 0; k < kMhaTile; k += 4) {
                        const float4 pk = *reinterpret_cast<const float4*>(p + k);
                        const float pv[4] = {pk.x, pk.y, pk.z, pk.w};
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const float2 v = lds2(sV + (k + u) * ld + c);
                            a0 = fmaf(pv[u], v.x, a0);
                            a1 = fmaf(pv[u], v.y, a1);
                        }
                    }
                    acc[rr][2 * j] = a0, acc[rr][2 * j + 1] = a1;
                }
            }
            __syncwarp();
        }
    }
#pragma unroll
    for (int rr = 0; rr < kRowsPerWarp; ++rr) {
        const int r = warp + 4 * rr;
        if (r >= x) break;
        const float inv = 1.f / l[rr];
#pragma unroll
        for (int j = 0; j < kPairs; ++j) {
            const int c = 2 * lane + 64 * j;
            if (c < d_k) {
                ctx[int64_t(b * x + r) * hk + i * d_k + c] = from_f32<T>(acc[rr][2 * j] * inv);
                ctx[int64_t(b * x + r) * hk + i * d_k + c + 1] = from_f32<T>(acc[rr][2 * j + 1] * inv);
            }
        }
    }
}

template <typename T>
void launch_mha_t(const void* Q, const void* Kc, const void* Vc, const int* npi, int B, int x, int h, int d_k,
                  int n_stride, float scale, void* ctx, cudaStream_t st) {
    const int ld = d_k + 16 / int(sizeof(T));
    const size_t smem = size_t(2) * 2 * kMhaTile * ld * sizeof(T) + sizeof(float) * (size_t(x) * d_k + 4 * kMhaTile);
    auto kern = mha_decode_kernel<T>;
    if (smem > 48 * 1024)
        ELA_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kern<<<dim3(B, h), kMhaThreads, smem, st>>>(static_cast<const T*>(Q), static_cast<const T*>(Kc),
                                                static_cast<const T*>(Vc), npi, B, x, h, d_k, n_stride,
                                                scale * 1.4426950408889634f, static_cast<T*>(ctx));
    ELA_CHECK_LAUNCH();
}

}  // namespace

bool mha_decode_supported(int x, int d_k, int dtype) {
    (void)dtype;  // rows are read 8 elements at a time
    return x >= 1 && x <= 16 && d_k >= 8 && d_k <= kMhaMaxDk && d_k % 8 == 0;
}

void launch_mha_decode(int dtype, const void* Q, const void* Kc, const void* Vc, const int* npi, int B, int x, int h,
                       int d_k, int n_stride, float scale, void* ctx, cudaStream_t st) {
    ELA_REQUIRE(mha_decode_supported(x, d_k, dtype), ELATTN_ERR_UNSUPPORTED,
                "MHA decode: x <= 16 rows per input, d_k a multiple of 8 up to 128");
    if (dtype == ELATTN_DTYPE_BF16)
        launch_mha_t<__nv_bfloat16>(Q, Kc, Vc, npi, B, x, h, d_k, n_stride, scale, ctx, st);
    else
        launch_mha_t<float>(Q, Kc, Vc, npi, B, x, h, d_k, n_stride, scale, ctx, st);
}

}  // namespace elattn_gpu
