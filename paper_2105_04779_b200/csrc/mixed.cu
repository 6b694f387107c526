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
// One CTA per (lane, head); scores of the generated rows staged in shared memory.
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

}  // namespace

void launch_mixed_combine(int dtype, const void* Q, const float2* stats, void* V, const void* Kc, const void* Vc,
                          int R, int h, int d_k, int64_t t_max, int t_out, const float* bk, float scale,
                          cudaStream_t st) {
    const float scale_log2 = scale * 1.4426950408889634f;
    const size_t smem = sizeof(float) * (size_t(d_k) * 3 + t_out);
    ELA_REQUIRE(smem <= 200u * 1024u, ELATTN_ERR_UNSUPPORTED, "mixed self-attention: generated cache too long");
    const unsigned grid = unsigned(int64_t(R) * h);
    if (dtype == ELATTN_DTYPE_BF16) {
        auto k = mixed_combine_kernel<__nv_bfloat16>;
        ELA_CHECK_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        k<<<grid, kThreads, smem, st>>>(static_cast<const __nv_bfloat16*>(Q), stats, static_cast<__nv_bfloat16*>(V),
                                        static_cast<const __nv_bfloat16*>(Kc), static_cast<const __nv_bfloat16*>(Vc), h,
                                        d_k, t_max, t_out, bk, scale_log2);
    } else {
        auto k = mixed_combine_kernel<float>;
        ELA_CHECK_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        k<<<grid, kThreads, smem, st>>>(static_cast<const float*>(Q), stats, static_cast<float*>(V),
                                        static_cast<const float*>(Kc), static_cast<const float*>(Vc), h, d_k, t_max,
                                        t_out, bk, scale_log2);
    }
    ELA_CHECK_LAUNCH();
}

}  // namespace elattn_gpu
