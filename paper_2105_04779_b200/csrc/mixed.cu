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
// One warp per (lane, head); scores of the generated rows staged in shared memory.
#include "common.cuh"
#include "kernels.h"

namespace elattn_gpu {

namespace {

constexpr int kWarps = 4;

template <typename T>
__global__ void __launch_bounds__(32 * kWarps) mixed_combine_kernel(const T* __restrict__ Q, const float2* __restrict__ stats,
                                                                    T* __restrict__ V, const T* __restrict__ Kc,
                                                                    const T* __restrict__ Vc, int R, int h, int d_k,
                                                                    int64_t t_max, int t_out,
                                                                    const float* __restrict__ bk, float scale_log2) {
    extern __shared__ float smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t row = int64_t(blockIdx.x) * kWarps + warp;  // r * h + i
    if (row >= int64_t(R) * h) return;
    const int i = int(row % h);
    float* sq = smem + warp * (d_k + t_out);  // Q_i, then the generated scores
    float* sc = sq + d_k;
    const T* q = Q + row * d_k;  // Q [R][h*d_k]: row r*h+i starts at (r*h+i)*d_k
    float sbias = 0.f;
    for (int d = lane; d < d_k; d += 32) {
        const float v = to_f32(q[d]);
        sq[d] = v;
        if (bk) sbias += v * bk[int64_t(i) * d_k + d];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sbias += __shfl_xor_sync(0xffffffffu, sbias, o);
    __syncwarp();
    const float2 st = stats[row];
    const float m_in = st.x + sbias * scale_log2, l_in = st.y;
    const T* Kr = Kc + row * t_max * d_k;  // cache [R][h][t_max][d_k]
    float mx = m_in;
    for (int r = lane; r < t_out; r += 32) {
        float g = 0.f;
        const T* k = Kr + int64_t(r) * d_k;
        for (int d = 0; d < d_k; ++d) g = fmaf(sq[d], to_f32(k[d]), g);
        g *= scale_log2;
        sc[r] = g;
        mx = fmaxf(mx, g);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float wg = 0.f;
    for (int r = lane; r < t_out; r += 32) {
        const float pr = exp2f(sc[r] - mx);
        sc[r] = pr;
        wg += pr;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wg += __shfl_xor_sync(0xffffffffu, wg, o);
    __syncwarp();
    const float w_in = l_in * exp2f(m_in - mx);
    const float inv_z = 1.f / (w_in + wg);
    const T* Vr = Vc + row * t_max * d_k;
    T* vo = V + row * d_k;
    for (int d = lane; d < d_k; d += 32) {
        float acc = 0.f;
        for (int r = 0; r < t_out; ++r) acc = fmaf(sc[r], to_f32(Vr[int64_t(r) * d_k + d]), acc);
        vo[d] = from_f32<T>((w_in * to_f32(vo[d]) + acc) * inv_z);
    }
}

}  // namespace

void launch_mixed_combine(int dtype, const void* Q, const float2* stats, void* V, const void* Kc, const void* Vc,
                          int R, int h, int d_k, int64_t t_max, int t_out, const float* bk, float scale,
                          cudaStream_t st) {
    const float scale_log2 = scale * 1.4426950408889634f;
    const size_t smem = sizeof(float) * size_t(kWarps) * (d_k + t_out);
    ELA_REQUIRE(smem <= 200u * 1024u, ELATTN_ERR_UNSUPPORTED, "mixed self-attention: generated cache too long");
    const unsigned grid = unsigned(ceil_div(int64_t(R) * h, kWarps));
    if (dtype == ELATTN_DTYPE_BF16) {
        auto k = mixed_combine_kernel<__nv_bfloat16>;
        ELA_CHECK_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        k<<<grid, 32 * kWarps, smem, st>>>(static_cast<const __nv_bfloat16*>(Q), stats, static_cast<__nv_bfloat16*>(V),
                                           static_cast<const __nv_bfloat16*>(Kc), static_cast<const __nv_bfloat16*>(Vc),
                                           R, h, d_k, t_max, t_out, bk, scale_log2);
    } else {
        auto k = mixed_combine_kernel<float>;
        ELA_CHECK_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        k<<<grid, 32 * kWarps, smem, st>>>(static_cast<const float*>(Q), stats, static_cast<float*>(V),
                                           static_cast<const float*>(Kc), static_cast<const float*>(Vc), R, h, d_k,
                                           t_max, t_out, bk, scale_log2);
    }
    ELA_CHECK_LAUNCH();
}

}  // namespace elattn_gpu
