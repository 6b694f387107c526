// beam.cu — device-side beam-search candidate selection: the
// candidate generation + ordering of beam_search (decoding.hpp:186-230).  For input b,
// every finite (parent i < roots, token t) gives lp_sum = live_lp[b][i] + lprobs[b][i][t];
// the k best are returned in the reference's candidate_better order (decoding.hpp:163-167:
// higher lp_sum first, then smaller token, then smaller parent).  EOS handling, the
// finished pool and termination stay with the caller (the model's search loop).
//
// Candidates are ranked by one 64-bit key (smaller = better): the order-preserving bits of
// lp_sum inverted, then token, then parent.  One CTA per input: each thread keeps a sorted
// local top-k of its strided slice; k rounds of a block-wide min-reduction merge them.
#include "common.cuh"
#include "kernels.h"

namespace elattn_gpu {

namespace {

constexpr int kBeamThreads = 256;
constexpr int kMaxK = 32;

__device__ __forceinline__ uint32_t ordered(float f) {  // monotonic float -> uint32
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float unordered(uint32_t o) {
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}

__global__ void __launch_bounds__(kBeamThreads) beam_topk_kernel(const float* __restrict__ lprobs,
                                                                 const float* __restrict__ live_lp, int lanes, int roots,
                                                                 int V, int k, int* __restrict__ parent,
                                                                 int* __restrict__ token, float* __restrict__ lp_sum) {
    const int b = blockIdx.x, tid = threadIdx.x;
    uint64_t top[kMaxK];
#pragma unroll
    for (int j = 0; j < kMaxK; ++j) top[j] = ~0ull;
    const int64_t total = int64_t(roots) * V;
    for (int64_t c = tid; c < total; c += kBeamThreads) {
        const int i = int(c / V), t = int(c % V);
        const float v = lprobs[(int64_t(b) * lanes + i) * V + t];
        if (!isfinite(v)) continue;
        const float s = live_lp[int64_t(b) * lanes + i] + v;
        const uint64_t key = (uint64_t(~ordered(s)) << 32) | (uint64_t(uint32_t(t)) << 8) | uint64_t(i);
        if (key >= top[k - 1]) continue;
        // insertion into the sorted local list (k <= kMaxK, fully unrolled compare-swap)
        uint64_t carry = key;
#pragma unroll
        for (int j = 0; j < kMaxK; ++j) {
            if (j < k && carry < top[j]) {
                const uint64_t tmp = top[j];
                top[j] = carry;
                carry = tmp;
            }
        }
    }
    // k rounds: the block-wide best of the threads' list heads; its owner pops it
    __shared__ uint64_t red[kBeamThreads / 32];
    int head = 0;
    for (int r = 0; r < k; ++r) {
        uint64_t cand = ~0ull;
#pragma unroll
        for (int j = 0; j < kMaxK; ++j)
            if (j == head) cand = top[j];
        uint64_t m = cand;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t other = __shfl_xor_sync(0xffffffffu, m, o);
            m = other < m ? other : m;
        }
        if ((tid & 31) == 0) red[tid >> 5] = m;
        __syncthreads();
        uint64_t best = red[0];
#pragma unroll
        for (int w = 1; w < kBeamThreads / 32; ++w) best = red[w] < best ? red[w] : best;
        __syncthreads();
        if (cand == best && best != ~0ull) ++head;  // keys are unique: exactly one owner
        if (tid == 0) {
            const int64_t o = int64_t(b) * k + r;
            if (best == ~0ull) {
                parent[o] = -1, token[o] = -1, lp_sum[o] = -INFINITY;
            } else {
                parent[o] = int(best & 0xffu);
                token[o] = int((best >> 8) & 0xffffffu);
                lp_sum[o] = unordered(~uint32_t(best >> 32));
            }
        }
    }
}

}  // namespace

void launch_beam_topk(const float* lprobs, const float* live_lp, int B, int lanes, int roots, int V, int k,
                      int* parent, int* token, float* lp_sum, cudaStream_t st) {
    ELA_REQUIRE(k >= 1 && k <= kMaxK, ELATTN_ERR_UNSUPPORTED, "beam_candidates: k must be in [1, 32]");
    ELA_REQUIRE(lanes >= 1 && lanes <= 256 && roots >= 1 && roots <= lanes, ELATTN_ERR_SHAPE,
                "beam_candidates: 1 <= roots <= lanes <= 256");
    ELA_REQUIRE(V >= 1 && V < (1 << 24), ELATTN_ERR_SHAPE, "beam_candidates: vocabulary must be < 2^24");
    beam_topk_kernel<<<B, kBeamThreads, 0, st>>>(lprobs, live_lp, lanes, roots, V, k, parent, token, lp_sum);
    ELA_CHECK_LAUNCH();
}

}  // namespace elattn_gpu
