// simt_kernels.cu — the fp32 (FFMA) path of the EL decode step.
//
// These kernels are the product for ELATTN_DTYPE_F32 (the reference's f32
// precision class, gated at 1e-5 relative): single-pass TF32 tensor cores
// cannot meet that bound, so fp32 runs on CUDA cores.  They also serve bf16
// shapes outside the tcgen05 kernels' envelope (e.g. the reference tests'
// d_m = 8..128, d_k = 3).  All accumulation is fp32.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace elattn_gpu {

// --------------------------------------------------------------------------
// Batched GEMM, C = alpha * A . B^T + bias  (B stored [N][K]).
// Replaces the reference's matmul triple loop (tensor.hpp:161-178) for the
// projections Y.Wq, Q_i.Wk_i^T, C_i.Wv_i, V.Wo (attention.hpp:205-206, 286).
// --------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) simt_gemm_kernel(GemmArgs g) {
    constexpr int BM = 64, BN = 64, BK = 16;
    __shared__ float As[BK][BM + 4];
    __shared__ float Bs[BK][BN + 4];
    const int z = blockIdx.z;
    const T* A = static_cast<const T*>(g.A) + z * g.sAz;
    const T* B = static_cast<const T*>(g.B) + z * g.sBz;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < g.K; k0 += BK) {
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            const int e = tid + l * 256;  // 0..1023
            const int r = e / BK, c = e % BK;
            const int gm = m0 + r, gn = n0 + r, gk = k0 + c;
            As[c][r] = (gm < g.M && gk < g.K) ? to_f32(A[gm * g.lda + gk]) : 0.f;
            Bs[c][r] = (gn < g.N && gk < g.K) ? to_f32(B[gn * g.ldb + gk]) : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < BK; ++k) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[k][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[k][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
    T* C = static_cast<T*>(g.C) + z * g.sCz;
    const float* bias = g.bias ? g.bias + z * g.sbz : nullptr;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int gm = m0 + ty * 4 + i;
        if (gm >= g.M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gn = n0 + tx * 4 + j;
            if (gn >= g.N) continue;
            float v = acc[i][j] * g.alpha;
            if (bias) v += bias[gn];
            C[gm * g.ldc + gn] = from_f32<T>(v);
        }
    }
}

void launch_simt_gemm(int dtype, const GemmArgs& g, cudaStream_t st) {
    dim3 grid(unsigned(ceil_div(g.N, 64)), unsigned(ceil_div(g.M, 64)), unsigned(g.Z));
    if (dtype == ELATTN_DTYPE_BF16)
        simt_gemm_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(g);
    else
        simt_gemm_kernel<float><<<grid, 256, 0, st>>>(g);
    ELA_CHECK_LAUNCH();
}

// --------------------------------------------------------------------------
// Key-bias scalars s_{r,i} = Q_{r,i} . bk_i (attention.hpp:208-212).
// --------------------------------------------------------------------------
template <typename T>
__global__ void key_bias_kernel(const T* Q, const float* bk, int R, int h, int d_k, float* s) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= R * h) return;
    const int r = idx / h, i = idx % h;
    float acc = 0.f;
    for (int c = 0; c < d_k; ++c) acc = fmaf(to_f32(Q[(int64_t)r * h * d_k + i * d_k + c]), bk[i * d_k + c], acc);
    s[idx] = acc;
}

void launch_key_bias_scalars(int dtype, const void* Q, const float* bk, int R, int h, int d_k,
                             float* s, cudaStream_t st) {
    const int total = R * h;
    const int blocks = int(ceil_div(total, 256));
    if (dtype == ELATTN_DTYPE_BF16)
        key_bias_kernel<<<blocks, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(Q), bk, R, h, d_k, s);
    else
        key_bias_kernel<<<blocks, 256, 0, st>>>(static_cast<const float*>(Q), bk, R, h, d_k, s);
    ELA_CHECK_LAUNCH();
}

// --------------------------------------------------------------------------
// SIMT fused EL decode (the core of el_attention_folded, attention.hpp:272-280):
// one CTA owns kSimtRows (8) EL-Q rows of one input and streams H_b in kSimtTile-row tiles
// through shared memory once, using each tile as both key and value:
//   S = q'.Hᵀ  -> online softmax (exp2, running max / sum) -> O += P.H.
// No per-head K/V and no beam-expanded H is ever formed.
// --------------------------------------------------------------------------
constexpr int kSimtRows = 8;   // query rows per CTA (two CTAs per SM at d_m 1024 fp32)
constexpr int kSimtTile = 16;  // H rows per tile

template <typename T, int CPT>
__global__ void __launch_bounds__(256) el_decode_simt_kernel(const T* __restrict__ qp,
                                                             const T* __restrict__ H,
                                                             const int* __restrict__ n_per_input,
                                                             int rows_per_input, int n_stride,
                                                             int d_m, float scale_log2,
                                                             T* __restrict__ ctx, float2* __restrict__ stats,
                                                             int splits, float* __restrict__ part_o,
                                                             float2* __restrict__ part_ml,
                                                             const int* __restrict__ h_index) {
    extern __shared__ float smem[];
    // padded rows: q rows 16 banks apart (+16), H rows 4 apart land 16 banks apart (+4), so
    // the two half-warps of the score phase never collide
    const int ldq = d_m + 16, ldh = d_m + 4;
    float* sq = smem;                                // [kSimtRows][d_m + 16]
    float* sh = sq + kSimtRows * ldq;                // [kSimtTile][d_m + 4]
    float* sp = sh + kSimtTile * ldh;                // [kSimtRows][kSimtTile]
    float* s_alpha = sp + kSimtRows * kSimtTile;     // [kSimtRows]
    float* s_l = s_alpha + kSimtRows;                // [kSimtRows]
    float* s_m = s_l + kSimtRows;                    // [kSimtRows]
    const int b = blockIdx.y, r0 = blockIdx.x * kSimtRows, tid = threadIdx.x;
    const int n = n_per_input ? n_per_input[b] : n_stride;
    const T* Hb = H + (int64_t)(h_index ? h_index[b] : b) * n_stride * d_m;  // slot-indexed caches
    const int64_t row_base = (int64_t)b * rows_per_input + r0;
    const int nrows = min(kSimtRows, rows_per_input - r0);

    if (n < 1 || n > n_stride) {  // ragged length out of contract: loud NaN rows
        for (int e = tid; e < nrows * d_m; e += 256)
            ctx[(row_base + e / d_m) * d_m + e % d_m] = from_f32<T>(__int_as_float(0x7fc00000));
        if (stats != nullptr && tid < nrows) stats[row_base + tid] = make_float2(__int_as_float(0x7fc00000), 0.f);
        return;
    }
    for (int e = tid; e < kSimtRows * d_m; e += 256) {
        const int r = e / d_m, c = e % d_m;
        sq[r * ldq + c] = r < nrows ? to_f32(qp[(row_base + r) * d_m + c]) : 0.f;
    }
    float acc[kSimtRows][CPT];
#pragma unroll
    for (int r = 0; r < kSimtRows; ++r)
#pragma unroll
        for (int c = 0; c < CPT; ++c) acc[r][c] = 0.f;
    // Score-thread mapping: 16 threads per query row, one H row each.
    const int sr = tid / kSimtTile, st_ = tid % kSimtTile;
    float m_run = -INFINITY, l_run = 0.f;  // valid in threads with st_ == 0 (replicated)

    // split z of `splits` takes tiles [z T / S, (z + 1) T / S) of the context (flash-decoding
    // style; the partial rows are combined by simt_merge_kernel)
    const int T_all = (n + kSimtTile - 1) / kSimtTile;
    const int t_beg = int((int64_t(blockIdx.z) * T_all) / splits) * kSimtTile;
    const int t_end = min(n, int((int64_t(blockIdx.z + 1) * T_all) / splits) * kSimtTile);
    if (tid < kSimtRows) s_m[tid] = -INFINITY, s_l[tid] = 0.f;
    for (int t0 = t_beg; t0 < t_end; t0 += kSimtTile) {
        __syncthreads();  // previous tile fully consumed
        for (int e = tid; e < kSimtTile * d_m; e += 256) {
            const int r = e / d_m, c = e % d_m;
            sh[r * ldh + c] = (t0 + r < n) ? to_f32(Hb[(int64_t)(t0 + r) * d_m + c]) : 0.f;
        }
        __syncthreads();
        // scores, register-blocked: warp w = one 4 (q rows) x 4 (H rows) block (2 x 4 blocks
        // cover 8 x 16), its 32 lanes split K (k = lane, lane + 32, ...): 8 shared loads per 16
        // FMAs; an xor-16 sum then a butterfly reduce-scatter over 16 lanes leaves lane s
        // (mod 16) with score (4 rb + s/4, 4 tb + s%4)
        {
            const int ks = tid & 31, pair = tid >> 5, rb = pair >> 2, tb = pair & 3;
            float acc_s[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) acc_s[i] = 0.f;
            const float* a = sq + (rb * 4) * ldq;
            const float* hh = sh + (tb * 4) * ldh;
#pragma unroll 4
            for (int k = ks; k < d_m; k += 32) {
                float qa[4], hb[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) qa[i] = a[i * ldq + k];
#pragma unroll
                for (int j = 0; j < 4; ++j) hb[j] = hh[j * ldh + k];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc_s[i * 4 + j] = fmaf(qa[i], hb[j], acc_s[i * 4 + j]);
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) acc_s[i] += __shfl_xor_sync(0xffffffffu, acc_s[i], 16);
#pragma unroll
            for (int w = 8; w >= 1; w >>= 1) {
                const bool upper = (ks & w) != 0;
#pragma unroll
                for (int i = 0; i < w; ++i) {
                    const float send = upper ? acc_s[i] : acc_s[i + w];
                    const float keep = upper ? acc_s[i + w] : acc_s[i];
                    acc_s[i] = keep + __shfl_xor_sync(0xffffffffu, send, w);
                }
            }
            if (ks < 16) sp[(rb * 4 + (ks >> 2)) * kSimtTile + tb * 4 + (ks & 3)] = acc_s[0];
        }
        __syncthreads();
        // softmax threads: 16 per query row (threads past kSimtRows rows idle along)
        const bool srow = sr < kSimtRows;
        float s = srow ? sp[sr * kSimtTile + st_] : 0.f;
        __syncthreads();  // sp is rewritten with P below
        s = (t0 + st_ < n) ? s * scale_log2 : -INFINITY;
        float mx = s;
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o, 16));
        const float m_new = fmaxf(m_run, mx);
        const float p = exp2f(s - m_new);
        float sum = p;
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o, 16);
        const float alpha = exp2f(m_run - m_new);  // 0 on the first tile
        l_run = l_run * alpha + sum;
        m_run = m_new;
        if (srow) sp[sr * kSimtTile + st_] = p;
        if (srow && st_ == 0) {
            s_alpha[sr] = alpha;
            s_l[sr] = l_run;
            s_m[sr] = m_run;
            if (splits == 1 && stats != nullptr && sr < nrows) stats[row_base + sr] = make_float2(m_run, l_run);
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < kSimtRows; ++r) {
            const float a = s_alpha[r];
#pragma unroll
            for (int c = 0; c < CPT; ++c) acc[r][c] *= a;
        }
#pragma unroll 4
        for (int t = 0; t < kSimtTile; ++t) {
            float hv[CPT];
#pragma unroll
            for (int c = 0; c < CPT; ++c) {
                const int col = tid + c * 256;
                hv[c] = col < d_m ? sh[t * ldh + col] : 0.f;
            }
#pragma unroll
            for (int r = 0; r < kSimtRows; ++r) {
                const float pr = sp[r * kSimtTile + t];
#pragma unroll
                for (int c = 0; c < CPT; ++c) acc[r][c] = fmaf(pr, hv[c], acc[r][c]);
            }
        }
    }
    __syncthreads();
    if (splits > 1) {  // unnormalised partial rows + {m, l} for the merge
        const int64_t prow = int64_t(blockIdx.z) * gridDim.y * rows_per_input + row_base;
        if (tid < nrows) part_ml[prow + tid] = make_float2(s_m[tid], s_l[tid]);
#pragma unroll
        for (int r = 0; r < kSimtRows; ++r) {
            if (r >= nrows) break;
#pragma unroll
            for (int c = 0; c < CPT; ++c) {
                const int col = tid + c * 256;
                if (col < d_m) part_o[(prow + r) * d_m + col] = acc[r][c];
            }
        }
        return;
    }
#pragma unroll
    for (int r = 0; r < kSimtRows; ++r) {
        if (r >= nrows) break;
        const float inv = 1.f / s_l[r];
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
            const int col = tid + c * 256;
            if (col < d_m) ctx[(row_base + r) * d_m + col] = from_f32<T>(acc[r][c] * inv);
        }
    }
}

// Combines the `splits` partial rows of the split SIMT decode: M = max m_s,
// w_s = 2^(m_s - M), L = sum l_s w_s, C = sum w_s O_s / L (stats {M, L}).  One CTA per row.
template <typename T>
__global__ void __launch_bounds__(256) simt_merge_kernel(const float* __restrict__ part_o,
                                                         const float2* __restrict__ part_ml, int splits,
                                                         int64_t total_rows, int rows_per_input,
                                                         const int* __restrict__ n_per_input, int n_stride,
                                                         int d_m, T* __restrict__ ctx, float2* __restrict__ stats) {
    const int64_t row = blockIdx.x;
    if (n_per_input != nullptr) {
        const int n = n_per_input[row / rows_per_input];
        if (n < 1 || n > n_stride) return;  // the decode wrote loud NaN rows
    }
    float M = -INFINITY;
    for (int s = 0; s < splits; ++s) M = fmaxf(M, part_ml[s * total_rows + row].x);
    float L = 0.f;
    for (int s = 0; s < splits; ++s) {
        const float2 ml = part_ml[s * total_rows + row];
        L += ml.y * exp2f(ml.x - M);
    }
    const float inv = 1.f / L;
    for (int col = threadIdx.x; col < d_m; col += 256) {
        float acc = 0.f;
        for (int s = 0; s < splits; ++s) {
            const float2 ml = part_ml[s * total_rows + row];
            acc += part_o[(s * total_rows + row) * d_m + col] * exp2f(ml.x - M);
        }
        ctx[row * d_m + col] = from_f32<T>(acc * inv);
    }
    if (stats != nullptr && threadIdx.x == 0) stats[row] = make_float2(M, L);
}

template <typename T, int CPT>
static void launch_decode_cpt(const void* qp, const void* H, const int* npi, int B, int rows,
                              int n_stride, int d_m, float scale_log2, void* ctx, cudaStream_t st,
                              float2* stats, const int* h_index) {
    const size_t smem =
        sizeof(float) * (size_t(kSimtRows) * (d_m + 16) + size_t(kSimtTile) * (d_m + 4) +
                         kSimtRows * kSimtTile + 3 * kSimtRows);
    auto kern = el_decode_simt_kernel<T, CPT>;
    ELA_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    // split the context over CTAs when (row blocks x inputs) leave more than a quarter of the
    // SMs idle (measured: B = 8 BART 0.96 -> 0.48 ms per layer; at B = 32, 128 blocks on 148
    // SMs, the partial rows cost more than the idle SMs)
    const int blocks = int(ceil_div(rows, kSimtRows)) * B;
    const int T_all = int(ceil_div(n_stride, kSimtTile));
    static const int sms = [] {
        int dev = 0, v = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    // two 8-row CTAs fit per SM
    int splits = 4 * blocks >= 3 * sms ? 1 : int(ceil_div(2 * sms, blocks));
    splits = std::max(1, std::min({splits, 8, T_all}));
    // partial rows of the split context: stream-ordered scratch, released on every path
    struct Parts {
        float* o = nullptr;
        float2* ml = nullptr;
        cudaStream_t st;
        ~Parts() {
            if (o) cudaFreeAsync(o, st);
            if (ml) cudaFreeAsync(ml, st);
        }
    } parts{nullptr, nullptr, st};
    const int64_t total_rows = int64_t(B) * rows;
    if (splits > 1) {
        ELA_CHECK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&parts.o),
                                       sizeof(float) * size_t(splits) * size_t(total_rows) * d_m, st));
        ELA_CHECK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&parts.ml),
                                       sizeof(float2) * size_t(splits) * size_t(total_rows), st));
    }
    dim3 grid(unsigned(ceil_div(rows, kSimtRows)), unsigned(B), unsigned(splits));
    kern<<<grid, 256, smem, st>>>(static_cast<const T*>(qp), static_cast<const T*>(H), npi, rows,
                                  n_stride, d_m, scale_log2, static_cast<T*>(ctx), stats, splits, parts.o, parts.ml,
                                  h_index);
    ELA_CHECK_LAUNCH();
    if (splits > 1) {
        simt_merge_kernel<T><<<unsigned(total_rows), 256, 0, st>>>(parts.o, parts.ml, splits, total_rows, rows, npi,
                                                                   n_stride, d_m, static_cast<T*>(ctx), stats);
        ELA_CHECK_LAUNCH();
    }
}

template <typename T>
static void launch_decode_t(const void* qp, const void* H, const int* npi, int B, int rows,
                            int n_stride, int d_m, float scale_log2, void* ctx, cudaStream_t st,
                            float2* stats, const int* h_index) {
    const int cpt = int(ceil_div(d_m, 256));
    switch (cpt) {
        case 1: return launch_decode_cpt<T, 1>(qp, H, npi, B, rows, n_stride, d_m, scale_log2, ctx, st, stats, h_index);
        case 2: return launch_decode_cpt<T, 2>(qp, H, npi, B, rows, n_stride, d_m, scale_log2, ctx, st, stats, h_index);
        case 3: return launch_decode_cpt<T, 3>(qp, H, npi, B, rows, n_stride, d_m, scale_log2, ctx, st, stats, h_index);
        case 4: return launch_decode_cpt<T, 4>(qp, H, npi, B, rows, n_stride, d_m, scale_log2, ctx, st, stats, h_index);
        case 5: return launch_decode_cpt<T, 5>(qp, H, npi, B, rows, n_stride, d_m, scale_log2, ctx, st, stats, h_index);
        case 6: return launch_decode_cpt<T, 6>(qp, H, npi, B, rows, n_stride, d_m, scale_log2, ctx, st, stats, h_index);
        default:
            throw Status{ELATTN_ERR_UNSUPPORTED, "SIMT decode supports d_m <= 1536"};
    }
}

void launch_el_decode_simt(int dtype, const void* qp, const void* H, const int* n_per_input,
                           int B, int rows_per_input, int n_stride, int d_m, float scale,
                           void* ctx, cudaStream_t st, float2* stats, const int* h_index) {
    const float scale_log2 = scale * 1.4426950408889634f;
    if (dtype == ELATTN_DTYPE_BF16)
        launch_decode_t<__nv_bfloat16>(qp, H, n_per_input, B, rows_per_input, n_stride, d_m,
                                       scale_log2, ctx, st, stats, h_index);
    else
        launch_decode_t<float>(qp, H, n_per_input, B, rows_per_input, n_stride, d_m, scale_log2,
                               ctx, st, stats, h_index);
}

}  // namespace elattn_gpu
