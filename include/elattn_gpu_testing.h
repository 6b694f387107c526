/*
 * elattn_gpu_testing.h — test hooks of libelattn_gpu.so (not part of the
 * reference-facing boundary).  They expose single internal kernels so the
 * tests can pin them in isolation against a torch fp32 reference.
 */
#ifndef ELATTN_GPU_TESTING_H_
#define ELATTN_GPU_TESTING_H_

#include <stdint.h>

#include "elattn_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

/* C[z][m][n] = alpha * sum_k A[z][m][k] * B[z][n][k] + bias[z][n]   (bf16 in/out,
 * fp32 accumulate).  kernel: 0 = SIMT, 1 = tcgen05 (UNSUPPORTED if the shape is
 * outside its envelope). */
int elattn_gpu_testing_gemm_bf16(const void* A, int64_t lda, int64_t sAz, const void* B, int64_t ldb,
                                 int64_t sBz, void* C, int64_t ldc, int64_t sCz, const float* bias,
                                 int64_t sbz, int M, int N, int K, int Z, float alpha, int kernel,
                                 elattn_stream_t stream);

/* Force the block shape of the tcgen05 GEMM family for every following bf16 projection
 * (tests sweep every instantiation; 0 = the automatic per-shape choice): bn in
 * {64, 128, 256} columns per tile, mt in {1, 2} 128-row m-subtiles per CTA sharing the
 * B slice, kbp in {1, 2} k-blocks of 64 per TMA box.  Combinations without an
 * instantiation make the next GEMM fail with ELATTN_ERR_UNSUPPORTED. */
int elattn_gpu_testing_gemm_config(int bn, int mt, int kbp);

/* Small-M split-K GEMM (a cluster of sk CTAs per 128 x 64 output tile, partials reduced
 * through DSMEM): sk in {2, 4, 8} forces it where the shape allows, 0 disables it, -1 =
 * automatic (default: used when the plain tile grid would fill less than half the SMs). */
int elattn_gpu_testing_gemm_splitk(int sk);

/* Fused small-batch query expansion (one launch: Q = Y.W_Q + b_Q reduced over a cluster of 4
 * CTAs, then q' = Q_i.W_K,i^T): 0 disables it, 1 forces it where the shape allows (bf16,
 * d_k = 64, up to 33 clusters of 4), -1 = automatic (up to 64 query rows). */
int elattn_gpu_testing_qexp_fused(int mode);

/* GEMM epilogue: 0 = coalesced st.global through a per-warp smem transpose, 1 = 128-row
 * TMA tensor stores, -1 = per shape (default: TMA stores for the write-bound q' expansion). */
int elattn_gpu_testing_gemm_epilogue(int tma);

/* Programmatic dependent launch of the step's kernels on (1, default) or off (0). */
int elattn_gpu_testing_set_pdl(int on);

/* Device buffer (>= 64 u64) receiving %globaltimer stamps of CTA 0 of every following
 * tcgen05 GEMM launch (setup, each k-step's operands landing, accumulator ready, epilogue
 * done); NULL disables tracing. */
int elattn_gpu_testing_set_gemm_trace(unsigned long long* trace);

/* The fp32 path's 3xTF32 tensor-core GEMM on fp32 operands (split into hi/lo inside):
 * C[z][m][n] = alpha * sum_k A[z][m][k] B[z][n][k] + bias[z][n]; with C_lo non-null the
 * output is written as (C, C_lo) = (tf32(C), C - tf32(C)).  K % 32 == 0. */
int elattn_gpu_testing_gemm_tf32x3(const float* A, int64_t lda, int64_t sAz, const float* B, int64_t ldb,
                                   int64_t sBz, float* C, float* C_lo, int64_t ldc, int64_t sCz,
                                   const float* bias, int64_t sbz, int M, int N, int K, int Z, float alpha,
                                   elattn_stream_t stream);

/* Stage (2) with an explicit kernel choice: 0 = SIMT, 1 = tcgen05. */
int elattn_gpu_testing_decode_bf16(const void* qprime, const void* H, const int* n_per_input, int B,
                                   int rows, int n, int d_m, float scale, void* ctx, int kernel,
                                   elattn_stream_t stream);

/* Schedule of the tcgen05 decode for every following launch: 0 = automatic, 1 = stream-K,
 * 2 = whole inputs strided over the clusters, 3 = tail-split.  With n_per_input the
 * automatic choice is ragged stream-K up to 8 inputs per cluster. */
int elattn_gpu_testing_decode_sched(int mode);

/* Device buffer (>= 2*32*64 + 2*grid u64, e.g. 8192) that receives clock64 stamps from
 * the first cluster of every following tcgen05 decode launch (events x 64 tiles per CTA),
 * then %globaltimer at entry and exit of every CTA; NULL disables tracing. */
int elattn_gpu_testing_set_decode_trace(unsigned long long* trace);

/* Measurement builds only (make EXTRA=-DELA_TIMELINE): every CTA of the projection GEMM,
 * fused query-expansion, decode and merge kernels launched afterwards appends a 32-byte
 * record {entry, after-PDL-wait, exit (%globaltimer ns), kind, block} at records[*count++]
 * (up to capacity; NULL records disables).  ELATTN_ERR_UNSUPPORTED in production builds. */
int elattn_gpu_testing_timeline(void* records, unsigned* count, unsigned capacity);

#ifdef __cplusplus
}
#endif

#endif
