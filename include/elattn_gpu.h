/*
 * elattn_gpu.h — C ABI of the B200-native EL-attention decode path.
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/proj/include/elattn/attention.hpp).  Plain pointers and
 * sizes only; no exceptions, no torch types.  Each entry point names the
 * reference function it replaces.  The C++ wrapper with the reference's exact
 * signatures (elattn::gpu::el_attention_folded(const Tensor&, ...)) lives in
 * include/elattn_gpu.hpp and is built on these calls; the Python host mirror is
 * paper_2105_04779_b200/attention.py.
 *
 * Conventions (reference semantics, SURVEY.md §8 "math contract"):
 *   - all matrices row-major;
 *   - folded query row   = ((b * g) + k) * h + i   (attention.hpp:296-302);
 *   - output row         = b * g + k              (attention.hpp:283-288);
 *   - H of input b lives at H + b * n_stride * d_m and is used as both key and
 *     value source; it is never projected, copied or beam-expanded;
 *   - "EL-Q" (q') has the reference meaning (q.Wq_i + bq_i).Wk_i^T WITHOUT the
 *     1/sqrt(d_k) factor; the decode kernel folds 1/sqrt(d_k)*log2(e) into the
 *     single FFMA that feeds exp2 in its online softmax;
 *   - the key-bias scalars s (attention.hpp:192-195) may be passed but are not
 *     applied: softmax is shift invariant (test_attention.cpp:260-271);
 *   - element type of every activation buffer (Y, q', H, out) is the params
 *     dtype: ELATTN_DTYPE_F32 (fp32 storage, FFMA arithmetic) or
 *     ELATTN_DTYPE_BF16 (bf16 storage, tcgen05 tensor cores, fp32 accumulate).
 *
 * Errors: every call returns an elattn_status_t; the message of the last failure
 * on the calling thread is elattn_gpu_last_error_message().  Status values map
 * 1:1 onto the reference exception types (errors.hpp:8-31).
 *
 * Streams: every compute call is stream-ordered and asynchronous; buffers are
 * device pointers owned by the caller.  A params handle is immutable after
 * creation and may be shared read-only across streams.  `workspace` may be
 * NULL (the library then allocates stream-ordered scratch with
 * cudaMallocAsync); otherwise it must hold elattn_gpu_workspace_size(...) bytes.
 */
#ifndef ELATTN_GPU_H_
#define ELATTN_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    ELATTN_OK = 0,
    ELATTN_ERR_SHAPE = 1,       /* ShapeError   errors.hpp:8-11  */
    ELATTN_ERR_PARAM = 2,       /* ParamError   errors.hpp:13-16 */
    ELATTN_ERR_STATE = 3,       /* StateError   errors.hpp:18-21 */
    ELATTN_ERR_NUMERIC = 4,     /* NumericError errors.hpp:33-36 */
    ELATTN_ERR_CUDA = 5,        /* CUDA runtime / launch failure  */
    ELATTN_ERR_OOM = 6,         /* device allocation failure      */
    ELATTN_ERR_UNSUPPORTED = 7  /* shape outside the kernels' envelope */
} elattn_status_t;

typedef enum { ELATTN_DTYPE_F32 = 0, ELATTN_DTYPE_BF16 = 1 } elattn_dtype_t;

typedef struct elattn_gpu_params_s* elattn_gpu_params_t;
typedef struct CUstream_st* elattn_stream_t; /* == cudaStream_t */

/* Library version and the sm_100a kernels compiled in. */
const char* elattn_gpu_version(void);

/* Message of the last failing call on this thread ("" if none). */
const char* elattn_gpu_last_error_message(void);

/*
 * Replaces: AttentionParams (attention.hpp:13-81) — validate() + the weights.
 * Host fp64 arrays in the reference's per-head layout:
 *   Wq, Wk, Wv: [h][d_m][d_k];  Wo: [h][d_k][d_m];  bq, bk, bv: [h][d_k];  bo: [d_m].
 * Weights are packed once to device in `dtype` as W_Q^T [h*d_k][d_m],
 * W_K [h][d_m][d_k], W_V^T [h][d_k][d_m], W_O^T [d_m][h*d_k] (every GEMM operand
 * K-major), with fp32 biases; bv is zeroed when include_value_bias == 0.
 * Errors: PARAM (h, d_m, d_k < 1; bad dtype), OOM, CUDA.
 */
int elattn_gpu_params_create(int h, int d_m, int d_k, int dtype, int include_key_bias,
                             int include_value_bias, const double* Wq, const double* Wk,
                             const double* Wv, const double* Wo, const double* bq,
                             const double* bk, const double* bv, const double* bo,
                             elattn_gpu_params_t* out);
int elattn_gpu_params_destroy(elattn_gpu_params_t params);
int elattn_gpu_params_info(elattn_gpu_params_t params, int* h, int* d_m, int* d_k, int* dtype);

/*
 * Replaces: build_el_query (attention.hpp:197-215) for R query rows at once
 * (g queries of B inputs, R = B*g), already in the folded layout of
 * fold_el_queries (attention.hpp:293-304).
 *   Y       [R][d_m]        query rows (dtype)
 *   qprime  [R*h][d_m]      EL-Q rows, row r*h + i (dtype)
 *   s       [R*h] float or NULL  key-bias scalars (Q_{r,i} . bk_i; 0 if the flag is off)
 * Errors: SHAPE (R < 1).
 */
int elattn_gpu_build_el_query(elattn_gpu_params_t params, const void* Y, int R, void* qprime,
                              float* s, void* workspace, size_t workspace_bytes,
                              elattn_stream_t stream);

/*
 * Replaces: el_attention_folded (attention.hpp:262-290), batched over B inputs.
 *   qprime       [B*g*h][d_m]   EL-Q rows (dtype), row ((b*g)+k)*h + i
 *   s            [B*g*h] float or NULL (accepted, not applied — see above)
 *   H            [B][n][d_m]    per-input hidden states (dtype)
 *   n_per_input  device int[B] or NULL: ragged context lengths, 1 <= n_b <= n
 *                (rows n_b..n-1 of H_b are ignored; an out-of-range n_b writes NaN rows)
 *   out          [B*g][d_m]     (dtype), row b*g + k
 * Errors: SHAPE (B, g < 1), STATE (n < 1, the reference's "empty context").
 */
int elattn_gpu_el_attention_folded(elattn_gpu_params_t params, const void* qprime, const float* s,
                                   const void* H, const int* n_per_input, int B, int g, int n,
                                   void* out, void* workspace, size_t workspace_bytes,
                                   elattn_stream_t stream);

/*
 * Replaces: one EL cross-attention sub-layer for a batch of lanes — the
 * reference's per-lane el_attention(yc, H, cross_attn) calls (model.hpp:373-377,
 * attention.hpp:239-257) for B inputs x x beams in one stream-ordered pass:
 *   (1) query expansion  Q = Y.W_Q + b_Q ; q'_{r,i} = Q_{r,i}.W_K,i^T
 *   (2) fused decode     P = softmax(q'.H_b^T / sqrt(d_k)) ; C = P.H_b  (H read once)
 *   (3) output proj.     out = concat_i(C_{r,i}.W_V,i + b_V,i).W_O + b_O
 *   Y [B*x][d_m], H [B][n][d_m], out [B*x][d_m] (dtype).
 * Errors: SHAPE (B, x < 1), STATE (n < 1).
 */
int elattn_gpu_el_attention_step(elattn_gpu_params_t params, const void* Y, const void* H,
                                 const int* n_per_input, int B, int x, int n, void* out,
                                 void* workspace, size_t workspace_bytes, elattn_stream_t stream);
/*
 * The same over SLOT-INDEXED states: input b attends over H[h_index[b]] of
 * H [h_slots][n][d_m] (device h_index[B]; the hidden-state caches of decoder-only
 * self-attention after a copy-on-fork reorder, elattn_gpu_cache_fork).  h_index = NULL
 * is elattn_gpu_el_attention_step.  Errors as above; SHAPE (h_slots < 1 with h_index).
 */
int elattn_gpu_el_attention_step_indexed(elattn_gpu_params_t params, const void* Y, const void* H,
                                         const int* n_per_input, const int* h_index, int h_slots, int B, int x,
                                         int n, void* out, void* workspace, size_t workspace_bytes,
                                         elattn_stream_t stream);

/*
 * Stage (2) alone — the fused flash-style pass of el_attention_folded
 * (attention.hpp:272-280: scores, softmax, P.H) without the output projection:
 *   qprime [B*rows][d_m], H [B][n][d_m]  ->  ctx [B*rows][d_m]   (dtype)
 * rows = query rows per input (g*h).  Exposed for stage-level timing and for
 * callers that fuse their own projection.
 */
int elattn_gpu_el_attention_decode(elattn_gpu_params_t params, const void* qprime, const void* H,
                                   const int* n_per_input, int B, int rows, int n, void* ctx,
                                   elattn_stream_t stream);

/* Scratch bytes needed by the calls above for (B inputs, g queries each, n). */
size_t elattn_gpu_workspace_size(elattn_gpu_params_t params, int B, int g, int n);

/*
 * Which decode kernel a (params, g) pair dispatches to:
 *   0 = SIMT (fp32 FFMA, or bf16 storage with fp32 FFMA),
 *   1 = tcgen05/TMEM/TMA fused decode (bf16, cluster of 2 CTAs per input),
 *   2 = 3xTF32 tcgen05 kind::tf32 (fp32 path: S = q'.H^T, softmax, P.H) for 16-byte aligned
 *       buffers (unaligned fp32 buffers fall back to 0).
 */
int elattn_gpu_decode_kernel_kind(elattn_gpu_params_t params, int g);

/*
 * Batched decoder step.  Replaces the reference's decoder-step loop
 * (model.hpp:357-385: for every lane, for every layer, el_attention(yc,
 * encoder_output, cross_attn) at :373-377; lanes iterated by decoding.hpp:259-260) for
 * all B*x lanes at once: out = layer_{L-1}( ... layer_0(Y) ... ), each layer an
 * elattn_gpu_el_attention_step over the SAME encoder states H (one per input, shared by
 * every layer, beam and head — EL's cache saving).  The L steps (query expansion, fused
 * decode, projections) are captured once into a CUDA graph on a private stream and
 * replayed by elattn_gpu_decoder_run, so a step costs one graph launch on the host.
 *   layers       L params handles (same h, d_m, d_k, dtype)
 *   H            [B][n][d_m] device, n_per_input device int[B] or NULL (as in _step)
 *   Y_in, out    [B*x][d_m] device buffers bound at creation: write Y_in, run, read out
 *                (out may alias Y_in)
 * create waits for all prior device work (cudaDeviceSynchronize) and runs one eager
 * warm-up step into internal scratch before capturing; run is stream-ordered on `stream`.
 * Errors: PARAM (null / mismatched layers), SHAPE, STATE (n < 1), OOM, CUDA.
 */
typedef struct elattn_gpu_decoder_s* elattn_gpu_decoder_t;
int elattn_gpu_decoder_create(const elattn_gpu_params_t* layers, int L, const void* H, const int* n_per_input,
                              int B, int x, int n, const void* Y_in, void* out, elattn_gpu_decoder_t* dec);
int elattn_gpu_decoder_run(elattn_gpu_decoder_t dec, elattn_stream_t stream);
int elattn_gpu_decoder_destroy(elattn_gpu_decoder_t dec);
/* our own kernels launched by one run (the graph's kernel nodes) */
int64_t elattn_gpu_decoder_kernels_per_run(elattn_gpu_decoder_t dec);

/*
 * Per-lane hidden-state caches for decoder-only EL self-attention (BASELINE config 4, the
 * "hidden-state-only cache").  A cache is caller-owned device
 * memory [lanes][n_max][d_m] (dtype) plus a device int[lanes] of lengths; attention over
 * it is elattn_gpu_el_attention_step(params, Y, cache, lengths, lanes, 1, n_max, ...).
 *   append: cache[l][len[l]] = Y[l], ++len[l]   (a full lane's length becomes n_max + 1,
 *           i.e. NaN rows on the next step — loud, like an out-of-range n_per_input)
 *   gather: DecoderState::gather_lanes (model.hpp:291-306) on the device: dst lane i =
 *           copy of src lane parent[i] (rows 0..len-1); parents may repeat; an out-of-range
 *           parent gives the lane length n_max + 1 (loud).  rows_hint = expected length
 *           (sizes the grid only).  src and dst must not overlap.
 */
int elattn_gpu_cache_append(void* cache, const void* Y, int* lengths, int lanes, int n_max, int d_m, int dtype,
                            elattn_stream_t stream);
int elattn_gpu_cache_gather(const void* src, const int* src_lengths, void* dst, int* dst_lengths,
                            const int* parent, int lanes_in, int lanes_out, int n_max, int d_m, int dtype,
                            int rows_hint, elattn_stream_t stream);
/*
 * Slot-indexed caches (copy on fork): lane i's history lives in slot lane_slot[i] of
 * cache [layers][slots][n_max][d_m]; lengths stay per lane, [layers][lanes].
 *   append_indexed: cache[lane_slot[i]][len[i]] = Y[i], ++len[i] (one layer's cache).
 *   fork: gather_lanes (model.hpp:291-306) over the slot map — new lane i continues lane
 *     parent[i]'s history.  The first new lane (lowest index) with a given parent takes
 *     over the parent's slot (no copy); every further child of that parent gets a slot no
 *     new lane owns and a copy of rows 0..len-1 in every layer.  So permute_lanes and
 *     keep_lanes copy nothing and a beam reorder copies one history per duplicated parent.
 *     Writes slot_out[lanes_out] and lengths_out[layers][lanes_out]; lanes_out <= slots;
 *     an out-of-range parent gives the lane a free slot and length n_max + 1 (loud).
 *     workspace: >= elattn_gpu_cache_fork_workspace(slots, lanes_in, lanes_out) bytes,
 *     16-byte aligned.  Stream-ordered, graph-capturable.
 */
int elattn_gpu_cache_append_indexed(void* cache, const void* Y, int* lengths, const int* lane_slot, int lanes,
                                    int n_max, int d_m, int dtype, elattn_stream_t stream);
size_t elattn_gpu_cache_fork_workspace(int slots, int lanes_in, int lanes_out);
int elattn_gpu_cache_fork(void* cache, int layers, int slots, int n_max, int d_m, int dtype,
                          const int* lengths_in, int* lengths_out, const int* slot_in, int* slot_out,
                          const int* parent, int lanes_in, int lanes_out, int rows_hint, void* workspace,
                          size_t workspace_bytes, elattn_stream_t stream);
/*
 * Whole-lane gather of fixed-size per-lane state (e.g. the K/V caches of the mixed form,
 * [R][h][t_max][d_k]): dst lane i = src lane parent[i], bytes_per_lane a multiple of 16;
 * an out-of-range parent fills the lane with NaN bytes.  gather_lanes / keep_lanes /
 * permute_lanes (model.hpp:291-325) are this with the parent list they imply.
 */
int elattn_gpu_lane_gather(const void* src, void* dst, const int* parent, int lanes_in, int lanes_out,
                           int64_t bytes_per_lane, elattn_stream_t stream);

/*
 * Decoder-only MIXED self-attention.  Replaces
 * mixed_self_attention(q, prefix_hidden, gen_cache, p) (attention.hpp:309-365) and
 * KvCache::append (:134-150) for B inputs x x lanes:
 *   kv_append: K_i = Y.Wk_i (+ bk_i), V_i = Y.Wv_i (+ bv_i) of every lane's row at position
 *              t of the generated-token caches Kc, Vc [R][h][t_max][d_k] (dtype), R = B*x.
 *   mixed:     EL scores over the prefix P [B][n][d_m] (shared by an input's x lanes,
 *              n_per_input ragged) and multi-head scores over each lane's t_out cached
 *              rows, one joint softmax, value bias split by the prefix mass; out [R][d_m].
 *              As in the reference's incremental step (model.hpp:365-367) the caller
 *              appends the current row first.  Workspace: elattn_gpu_mixed_workspace_size.
 * Errors: SHAPE, STATE (empty prefix, t_out > t_max, append past t_max), PARAM.
 */
int elattn_gpu_kv_append(elattn_gpu_params_t params, const void* Y, int R, void* Kc, void* Vc, int t_max, int t,
                         elattn_stream_t stream);
int elattn_gpu_mixed_self_attention(elattn_gpu_params_t params, const void* Y, const void* P, const int* n_per_input,
                                    int B, int x, int n, const void* Kc, const void* Vc, int t_max, int t_out,
                                    void* out, void* workspace, size_t workspace_bytes, elattn_stream_t stream);
size_t elattn_gpu_mixed_workspace_size(elattn_gpu_params_t params, int B, int x);

/*
 * Multi-head-attention baseline with per-head K/V caches, on the
 * library's own kernels: the reference's multi_head_attention (attention.hpp:96-113) for
 * B inputs x x query rows at once, split as KvCache construction + attention_over_cache
 * (:118-180).  It is the comparator EL-attention is measured against on the same GPU.
 *   mha_kv_build: Kc, Vc [h][B][n][d_k] (dtype) <- K_i = H.W_K,i (+ b_K,i if
 *                 include_key_bias), V_i = H.W_V,i (+ b_V,i if include_value_bias), for every
 *                 position of every input H [B][n][d_m].
 *   mha_attention: out[b*x + k] = sum_i softmax(Q_{b,k,i} . K_i(b)^T / sqrt(d_k)) . V_i(b)
 *                 . W_O,i + b_O with Q = Y.W_Q + b_Q; Y, out [B*x][d_m]; n_per_input (device
 *                 int[B] or NULL) masks positions >= n_b of input b's cache (stride n).
 *                 x <= 16; d_k a multiple of 8 up to 128.
 *                 Workspace: elattn_gpu_mha_workspace_size (or NULL: stream-ordered alloc).
 */
int elattn_gpu_mha_kv_build(elattn_gpu_params_t params, const void* H, int B, int n, void* Kc, void* Vc,
                            elattn_stream_t stream);
size_t elattn_gpu_mha_workspace_size(elattn_gpu_params_t params, int B, int x);
int elattn_gpu_mha_attention(elattn_gpu_params_t params, const void* Y, const void* Kc, const void* Vc,
                             const int* n_per_input, int B, int x, int n, void* out, void* workspace,
                             size_t workspace_bytes, elattn_stream_t stream);

/*
 * Beam-search candidate selection on the device (decoding.hpp:186-230).
 * For each input b: candidates (parent i < roots, token t) with lp_sum = live_lp[b*lanes+i]
 * + lprobs[(b*lanes+i)*V + t], non-finite log-probs skipped; the k best (k <= 32) in the
 * reference's candidate_better order (decoding.hpp:163-167: higher lp_sum, then smaller
 * token, then smaller parent) -> parent/token/lp_sum [B][k] (parent -1 when fewer than k).
 * roots = 1 on the first step (all lanes identical), = lanes afterwards.  penalty (may be
 * NULL): device float[B][V] >= 0 subtracted from every finite log-prob before the sum (the
 * raw-log-prob pre-filter is exact only for non-negative penalties: negative values are
 * outside the contract; the Python wrapper rejects them) —
 * diverse_beam_search's `v -= strength * step_token_counts[tok]` (decoding.hpp:312-316),
 * called once per group with that group's contiguous lanes.
 */
int elattn_gpu_beam_candidates(const float* lprobs, const float* live_lp, const float* penalty, int B, int lanes,
                               int roots, int V, int k, int* parent, int* token, float* lp_sum,
                               elattn_stream_t stream);

/* Device-kernel launches issued by this thread since the last reset (for bench
 * accounting of gpu_launches). */
int64_t elattn_gpu_launch_count(void);
void elattn_gpu_reset_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* ELATTN_GPU_H_ */
