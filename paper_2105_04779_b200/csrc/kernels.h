// kernels.h — host-side launchers for every device kernel in the library.
#pragma once

#include <algorithm>

#include <cuda_runtime.h>

#include <cstdint>

namespace elattn_gpu {

// Batched GEMM on CUDA cores (fp32 FFMA), operands of storage type `dtype`:
//   C[z][m][n] = alpha * sum_k A[z][m][k] * B[z][n][k] + bias[z][n]
// (B is given K-major, i.e. as [N][K]).  bias may be null; C has the same
// storage dtype as A/B unless c_f32.
struct GemmArgs {
    const void* A;
    int64_t lda, sAz;
    const void* B;
    int64_t ldb, sBz;
    void* C;
    int64_t ldc, sCz;
    const float* bias;
    int64_t sbz;
    int M, N, K, Z;
    float alpha;
    int b_static = 0;  // 1: B (the weights) is never written by a kernel of the stream: the GEMM may
                       // fetch it before its programmatic-dependent-launch wait
    int c_keep = 0;    // 1: keep C in L2 (evict-last stores): the next kernel reads it back
};
void launch_simt_gemm(int dtype, const GemmArgs& g, cudaStream_t st);

// s[r*h + i] = sum_c Q[r][i*d_k + c] * bk[i*d_k + c]  (key-bias scalars).
void launch_key_bias_scalars(int dtype, const void* Q, const float* bk, int R, int h, int d_k,
                             float* s, cudaStream_t st);

// SIMT fused EL decode: ctx[b*rows + r] = softmax(q'_r . H_b^T * scale) . H_b.
// stats (optional, may be null): per query row float2 {m, l} of the softmax in log2
// units — p_j = 2^(s_j * scale * log2(e) - m) / l — for callers that merge the decode
// with other score sources (mixed self-attention).
void launch_el_decode_simt(int dtype, const void* qp, const void* H, const int* n_per_input,
                           int B, int rows_per_input, int n_stride, int d_m, float scale,
                           void* ctx, cudaStream_t st, float2* stats = nullptr, const int* h_index = nullptr);

// tcgen05 GEMM family (tc_gemm.cu: bf16 in, fp32 accumulate in TMEM, bf16 out), same
// contract as launch_simt_gemm but requires K % 64 == 0, 16-byte aligned rows and
// N % 16 == 0.  tc_gemm_supported returns false outside that envelope.
bool tc_gemm_supported(const GemmArgs& g);
// Fused small-batch query expansion q' = (Y.W_Q + b_Q)_i . W_K,i^T (bf16; one launch, cluster
// of 4 CTAs per 128-row tile and head); returns false when the shape is outside its envelope.
bool tc_qexp_fused(const void* Y, int M, const void* WqT, const float* bq, const void* Wk, void* qp, int h, int d_m,
                   int d_k, cudaStream_t st);
void launch_tc_gemm(const GemmArgs& g, cudaStream_t st);

// Testing / tuning override of the tcgen05 GEMM block shape (0 = automatic choice).
extern int g_decode_sched_override;
extern int g_qexp_fused;
extern int g_gemm_force_bn, g_gemm_force_mt, g_gemm_force_kbp, g_gemm_force_splitk;
extern unsigned long long* g_gemm_trace;
extern int g_gemm_epilogue_tma;

// fp32 path on the tensor cores (tf32_gemm.cu): 3xTF32 GEMM
//   C[z][m][n] = alpha * sum_k (A_hi B_hi + A_hi B_lo + A_lo B_hi) + bias[z][n]
// A [z][m][k], B [z][n][k] (both K-major); C fp32, written as (C, C_lo) = (tf32(C),
// C - tf32(C)) when C_lo != null.  K % 32 == 0.
struct Tf32GemmArgs {
    const float* A_hi;
    const float* A_lo;
    int64_t lda, sAz;
    const float* B_hi;
    const float* B_lo;
    int64_t ldb, sBz;
    float* C;
    float* C_lo;
    int64_t ldc, sCz;
    const float* bias;
    int64_t sbz;
    int M, N, K, Z;
    float alpha;
};
bool tf32_gemm_supported(const Tf32GemmArgs& g);
void launch_tf32_gemm(const Tf32GemmArgs& g, cudaStream_t st);
// X [rows][cols] (row stride ld) -> hi, lo [rows][cols]; rows r with npi and
// r % n_stride >= npi[r / n_stride] are zeroed; h_index: output block b of n_stride rows
// reads block h_index[b] of X (slot-indexed caches)
void launch_tf32_split(const float* X, int64_t rows, int cols, int64_t ld, float* hi, float* lo, const int* npi,
                       int n_stride, cudaStream_t st, const int* h_index = nullptr);
// H [B][n][d_m] -> transposed hi/lo [B][d_m][n_pad], keys >= n_b (npi) or >= n zeroed;
// input b reads H[h_index[b]] when h_index is given
void launch_tf32_split_t(const float* H, int B, int n, int d_m, int n_pad, const int* npi, float* hi, float* lo,
                         cudaStream_t st, const int* h_index = nullptr);
// softmax over the first n_b of each score row (see tf32_gemm.cu) -> (P_hi, P_lo), stats
void launch_tf32_softmax(const float* S, int64_t total_rows, int rows, int n_stride, int ld, const int* npi,
                         float scale, float* P_hi, float* P_lo, float2* stats, cudaStream_t st);

// MHA baseline decode over per-input K/V caches [h][B][n_stride][d_k] (mha.cu).
bool mha_decode_supported(int x, int d_k, int dtype);
void launch_mha_decode(int dtype, const void* Q, const void* Kc, const void* Vc, const int* npi, int B, int x, int h,
                       int d_k, int n_stride, float scale, void* ctx, cudaStream_t st);

// Mixed self-attention merge (mixed.cu): see the file header.
void launch_mixed_combine(int dtype, const void* Q, const float2* stats, void* V, const void* Kc, const void* Vc,
                          int R, int h, int d_k, int64_t t_max, int t_out, const float* bk, float scale,
                          cudaStream_t st);

// Beam-search candidate selection (beam.cu).
int beam_splits(int B, int V);
void launch_beam_topk(const float* lprobs, const float* live_lp, const float* penalty, int B, int lanes, int roots,
                      int V, int k,
                      uint64_t* part, int splits, int* parent, int* token, float* lp_sum, cudaStream_t st);

// Per-lane hidden-state caches (lane_cache.cu).
void launch_lane_gather(const void* src, void* dst, const int* parent, int lanes_in, int lanes_out,
                        int64_t bytes_per_lane, cudaStream_t st);
void launch_cache_append(void* cache, const void* Y, int* len, int lanes, int n_max, int d_m, int dtype,
                         cudaStream_t st, const int* lane_slot = nullptr);
// slot-indexed caches: copy-on-fork reorder (see lane_cache.cu)
size_t cache_fork_workspace(int slots, int lanes_in, int lanes_out);
void launch_cache_fork(void* cache, int layers, int slots, int n_max, int d_m, int dtype, const int* len_in,
                       int* len_out, const int* slot_in, int* slot_out, const int* parent, int lanes_in, int lanes_out,
                       int rows_hint, void* ws, size_t ws_bytes, cudaStream_t st);
void launch_cache_gather(const void* src, const int* src_len, void* dst, int* dst_len, const int* parent,
                         int lanes_in, int lanes_out, int n_max, int d_m, int dtype, int rows_hint,
                         cudaStream_t st);

// Testing hook: when non-null, the tcgen05 decode writes clock64 stamps of its
// first cluster: trace[(cta*24 + event)*64 + tile].
extern unsigned long long* g_decode_trace;
// measurement builds (-DELA_TIMELINE, timeline.cuh): per-CTA step timeline buffers of the
// GEMM and decode translation units (false when the build has no timeline)
struct TlRec;
bool tl_set_gemm(TlRec* buf, unsigned* cnt, unsigned cap);
bool tl_set_decode(TlRec* buf, unsigned* cnt, unsigned cap);

// tcgen05/TMA fused EL decode for bf16 (cluster of 2 CTAs per input, split d_m).
bool el_decode_tc_supported(int rows_per_input, int d_m);
// `part`: scratch of el_decode_tc_scratch_bytes(d_m) bytes for the partial records of
// inputs split across clusters (stream-ordered, owned by the caller's workspace).
size_t el_decode_tc_scratch_bytes(int d_m);
void launch_el_decode_tc(const void* qp, const void* H, const int* n_per_input, int B,
                         int rows_per_input, int n_stride, int d_m, float scale, void* ctx,
                         cudaStream_t st, float2* stats, float* part, bool h_static = false,
                         const int* h_index = nullptr, int h_slots = 0);

}  // namespace elattn_gpu
