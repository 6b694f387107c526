// mixed.cu — decoder-only MIXED self-attention on the GPU (reference mixed_self_attention,
// attention.hpp:309-365): EL scores over the prefix hidden states shared by an input's
// lanes, multi-head scores over each lane's generated-token K/V cache (KvCache,
// :118-150), ONE joint softmax.
//
// The prefix part runs through the fused EL decode, which also emits each row's softmax
// statistics {m, l} (log2 units); the V projection then gives V_in = C_in.Wv_i + bv_i.
// This kernel scores the generated part and merges the two halves of the joint softmax:
//   m'_in = m_in + s_i (s_i = Q_i.bk_i, the key-bias term the decode leaves out; K rows
//           of the cache carry bk, so both parts then share the reference's shift)
//   M = max(m'_in, max_r g_r),  g_r = Q_i.K_r * scale * log2(e)
//   w_in = l_in 2^(m'_in - M),  p_r = 2^(g_r - M),  Z = w_in + sum_r p_r
//   V_i <- (w_in V_in,i + sum_r p_r V_r) / Z
// which is the reference's prefix head with the value bias scaled by the prefix mass plus
// the cached head (values already biased) — the output projection follows unchanged.
// One CTA per (lane, head); scores of the generated rows staged in shared memory (the
// vectorised kernel below for the usual head widths, the scalar one otherwise).
#include "common.cuh"
#include "kernels.h"

namespace elattn_gpu {

namespace {

constexpr int kThreads = 128;

__device__ __forceinline__ float block_reduce_max(float v, float* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    v = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
    __syncthreads();
    return v;
}
__device__ __forceinline__ float block_reduce_sum(float v, float* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    v = red[0] + red[1] + red[2] + red[3];
    __syncthreads();
    return v;
}

// 8 consecutive elements as fp32
__device__ __forceinline__ void load8(const __nv_bfloat16* p, float (&o)[8]) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(h[i]);
        o[2 * i] = f.x, o[2 * i + 1] = f.y;
    }
}
__device__ __forceinline__ void load8(const float* p, float (&o)[8]) {
    const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
    o[0] = a.x, o[1] = a.y, o[2] = a.z, o[3] = a.w, o[4] = b.x, o[5] = b.y, o[6] = b.z, o[7] = b.w;
}

// One CTA (128 threads) per (lane r, head i).  Scores: thread per cached row (rows staged
// 16 bytes at a time); context: thread per (dimension, row parity) with coalesced row reads.
template <typename T>
__global__ void __launch_bounds__(kThreads) mixed_combine_kernel(const T* __restrict__ Q, const float2* __restrict__ stats,
                                                                 T* __restrict__ V, const T* __restrict__ Kc,
                                                                 const T* __restrict__ Vc, int h, int d_k, int64_t t_max,
                                                                 int t_out, const float* __restrict__ bk,
                                                                 float scale_log2) {
    extern __shared__ float smem[];
    float* sq = smem;            // Q_i [d_k]
    float* sc = sq + d_k;        // generated-row scores / probabilities [t_out]
    float* acc2 = sc + t_out;    // [2][d_k] partial contexts (row parity)
    __shared__ float red[4];
    const int64_t row = blockIdx.x;  // r * h + i
    const int i = int(row % h), tid = int(threadIdx.x);
    const T* q = Q + row * d_k;  // Q [R][h*d_k]: row r*h+i starts at (r*h+i)*d_k
    float sb = 0.f;
    for (int d = tid; d < d_k; d += kThreads) {
        const float v = to_f32(q[d]);
        sq[d] = v;
        if (bk) sb += v * bk[int64_t(i) * d_k + d];
    }
    __syncthreads();
    const float sbias = bk ? block_reduce_sum(sb, red) : 0.f;
    const float2 st = stats[row];
    const float m_in = st.x + sbias * scale_log2, l_in = st.y;
    const T* Kr = Kc + row * t_max * d_k;  // cache [R][h][t_max][d_k]
    const bool vec = (d_k % 8) == 0;
    float mx = m_in;
    for (int r = tid; r < t_out; r += kThreads) {
        const T* k = Kr + int64_t(r) * d_k;
        float g = 0.f;
        if (vec) {
            for (int d = 0; d < d_k; d += 8) {
                float kv[8];
                load8(k + d, kv);
#pragma unroll
                for (int e = 0; e < 8; ++e) g = fmaf(sq[d + e], kv[e], g);
            }
        } else {
            for (int d = 0; d < d_k; ++d) g = fmaf(sq[d], to_f32(k[d]), g);
        }
        g *= scale_log2;
        sc[r] = g;
        mx = fmaxf(mx, g);
    }
    mx = block_reduce_max(mx, red);
    float wg = 0.f;
    for (int r = tid; r < t_out; r += kThreads) {
        const float pr = exp2f(sc[r] - mx);
        sc[r] = pr;
        wg += pr;
    }
    wg = block_reduce_sum(wg, red);  // (its barriers also publish sc[])
    const float w_in = l_in * exp2f(m_in - mx);
    const float inv_z = 1.f / (w_in + wg);
    const T* Vr = Vc + row * t_max * d_k;
    for (int e = tid; e < 2 * d_k; e += kThreads) {  // (dimension d, row parity)
        const int d = e % d_k, par = e / d_k;
        float a = 0.f;
#pragma unroll 4
        for (int r = par; r < t_out; r += 2) a = fmaf(sc[r], to_f32(Vr[int64_t(r) * d_k + d]), a);
        acc2[par * d_k + d] = a;
    }
    __syncthreads();
    T* vo = V + row * d_k;
    for (int d = tid; d < d_k; d += kThreads)
        vo[d] = from_f32<T>((w_in * to_f32(vo[d]) + acc2[d] + acc2[d_k + d]) * inv_z);
}

// Vectorised form (d_k in {8, 16, 32, 64, 128}): the 128 threads are RG row groups x CG = d_k / 8
// column groups; every thread moves 8 consecutive dimensions of a cached row with one 16-byte
// load (a row is CG threads, RG rows per pass, all loads coalesced), score dot products are
// reduced over the CG lanes of a row with shuffles, and the context accumulates 8 dimensions
// per thread, reduced over the row groups once through shared memory.
template <typename T, int CG>
__global__ void __launch_bounds__(kThreads) mixed_combine_vec_kernel(const T* __restrict__ Q, const float2* __restrict__ stats,
                                                                     T* __restrict__ V, const T* __restrict__ Kc,
                                                                     const T* __restrict__ Vc, int h, int64_t t_max,
                                                                     int t_out, const float* __restrict__ bk,
                                                                     float scale_log2) {
    constexpr int d_k = 8 * CG, RG = kThreads / CG;
    extern __shared__ float smem[];
    float* sc = smem;            // generated-row scores / probabilities [t_out]
    float* part = sc + t_out;    // [RG][d_k] partial contexts
    __shared__ float red[4];
    const int64_t row = blockIdx.x;  // r * h + i
    const int i = int(row % h), tid = int(threadIdx.x), g = tid / CG, c = tid % CG;
    float q[8];
    load8(Q + row * d_k + 8 * c, q);
    float sb = 0.f;
    if (bk != nullptr && g == 0) {
#pragma unroll
        for (int e = 0; e < 8; ++e) sb += q[e] * bk[int64_t(i) * d_k + 8 * c + e];
    }
    const float sbias = bk ? block_reduce_sum(sb, red) : 0.f;
    const float2 st = stats[row];
    const float m_in = st.x + sbias * scale_log2, l_in = st.y;
    const T* Kr = Kc + row * t_max * d_k + 8 * c;  // cache [R][h][t_max][d_k]
    float mx = m_in;
    for (int r0 = 0; r0 < t_out; r0 += RG) {
        const int r = r0 + g;
        float dot = 0.f;
        if (r < t_out) {
            float kv[8];
            load8(Kr + int64_t(r) * d_k, kv);
#pragma unroll
            for (int e = 0; e < 8; ++e) dot = fmaf(q[e], kv[e], dot);
        }
#pragma unroll
        for (int o = CG / 2; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        if (r < t_out) {
            const float gs = dot * scale_log2;
            if (c == 0) sc[r] = gs;
            mx = fmaxf(mx, gs);
        }
    }
    mx = block_reduce_max(mx, red);  // (its barriers also publish sc[])
    float wg = 0.f;
    for (int r = tid; r < t_out; r += kThreads) {
        const float pr = exp2f(sc[r] - mx);
        sc[r] = pr;
        wg += pr;
    }
    wg = block_reduce_sum(wg, red);
    const float w_in = l_in * exp2f(m_in - mx);
    const float inv_z = 1.f / (w_in + wg);
    const T* Vr = Vc + row * t_max * d_k + 8 * c;
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.f;
#pragma unroll 2
    for (int r = g; r < t_out; r += RG) {
        float vv[8];
        load8(Vr + int64_t(r) * d_k, vv);
        const float pr = sc[r];
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = fmaf(pr, vv[e], acc[e]);
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) part[g * d_k + 8 * c + e] = acc[e];
    __syncthreads();
    T* vo = V + row * d_k;
    for (int d = tid; d < d_k; d += kThreads) {
        float a = 0.f;
        for (int gg = 0; gg < RG; ++gg) a += part[gg * d_k + d];  // fixed order: deterministic
        vo[d] = from_f32<T>((w_in * to_f32(vo[d]) + a) * inv_z);
    }
}

template <typename T>
void launch_combine_typed(const void* Q, const float2* stats, void* V, const void* Kc, const void* Vc, int R, int h,
                          int d_k, int64_t t_max, int t_out, const float* bk, float scale_log2, cudaStream_t st) {
    const unsigned grid = unsigned(int64_t(R) * h);
    auto go = [&](auto kern, size_t smem) {
        ELA_REQUIRE(smem <= 200u * 1024u, ELATTN_ERR_UNSUPPORTED, "mixed self-attention: generated cache too long");
        ELA_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        kern<<<grid, kThreads, smem, st>>>(static_cast<const T*>(Q), stats, static_cast<T*>(V), static_cast<const T*>(Kc),
                                           static_cast<const T*>(Vc), h, t_max, t_out, bk, scale_log2);
    };
    const size_t vsmem = sizeof(float) * (size_t(t_out) + size_t(kThreads) * 8);  // sc + [RG][d_k] = 128 x 8
    const bool aligned = (reinterpret_cast<uintptr_t>(Q) | reinterpret_cast<uintptr_t>(Kc) |
                          reinterpret_cast<uintptr_t>(Vc)) % 16 == 0;
    if (aligned) {
        switch (d_k) {
            case 8: return go(mixed_combine_vec_kernel<T, 1>, vsmem);
            case 16: return go(mixed_combine_vec_kernel<T, 2>, vsmem);
            case 32: return go(mixed_combine_vec_kernel<T, 4>, vsmem);
            case 64: return go(mixed_combine_vec_kernel<T, 8>, vsmem);
            case 128: return go(mixed_combine_vec_kernel<T, 16>, vsmem);
            default: break;
        }
    }
    const size_t smem = sizeof(float) * (size_t(d_k) * 3 + t_out);
    ELA_REQUIRE(smem <= 200u * 1024u, ELATTN_ERR_UNSUPPORTED, "mixed self-attention: generated cache too long");
    auto k = mixed_combine_kernel<T>;
    ELA_CHECK_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    k<<<grid, kThreads, smem, st>>>(static_cast<const T*>(Q), stats, static_cast<T*>(V), static_cast<const T*>(Kc),
                                    static_cast<const T*>(Vc), h, d_k, t_max, t_out, bk, scale_log2);
}

}  // namespace

void launch_mixed_combine(int dtype, const void* Q, const float2* stats, void* V, const void* Kc, const void* Vc,
                          int R, int h, int d_k, int64_t t_max, int t_out, const float* bk, float scale,
                          cudaStream_t st) {
    const float scale_log2 = scale * 1.4426950408889634f;
    if (dtype == ELATTN_DTYPE_BF16)
        launch_combine_typed<__nv_bfloat16>(Q, stats, V, Kc, Vc, R, h, d_k, t_max, t_out, bk, scale_log2, st);
    else
        launch_combine_typed<float>(Q, stats, V, Kc, Vc, R, h, d_k, t_max, t_out, bk, scale_log2, st);
    ELA_CHECK_LAUNCH();
}

}  // namespace elattn_gpu
