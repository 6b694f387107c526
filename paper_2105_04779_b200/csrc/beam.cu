// beam.cu — device-side beam-search candidate selection: the
// candidate generation + ordering of beam_search (decoding.hpp:186-230).  For input b,
// every finite (parent i < roots, token t) gives lp_sum = live_lp[b][i] + lprobs[b][i][t];
// the k best are returned in the reference's candidate_better order (decoding.hpp:163-167:
// higher lp_sum first, then smaller token, then smaller parent).  An optional per-input
// token penalty (>= 0, so the float4 pre-filter on the raw log-probs stays a necessary
// condition) is subtracted from each finite log-prob first: diverse beam search's
// `v -= strength * step_token_counts[tok]` (decoding.hpp:312-316), one call per group.
// EOS handling, the finished pool and termination stay with the caller (the search loop).
//
// Candidates are ranked by one 64-bit key (smaller = better): the order-preserving bits of
// lp_sum inverted, then token, then parent.  Phase 1: CTAs (column split, input) scan their
// slice; each warp keeps a lane-distributed sorted top-k (ballot-filtered against its k-th
// key, so after the first few hundred candidates almost nothing is inserted); phase 2: one
// warp per input merges the splits' lists and decodes the keys.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace elattn_gpu {

namespace {

constexpr int kBeamThreads = 256;
constexpr int kBeamWarps = kBeamThreads / 32;
constexpr int kMaxK = 32;
constexpr int kUnroll = 4;

__device__ __forceinline__ uint32_t ordered(float f) {  // monotonic float -> uint32
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float unordered(uint32_t o) {
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}
__device__ __forceinline__ uint64_t rank_key(float s, int t, int i) {
    return (uint64_t(~ordered(s)) << 32) | (uint64_t(uint32_t(t)) << 8) | uint64_t(i);
}

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint64_t umax64(uint64_t a, uint64_t b) { return a < b ? b : a; }

// Ascending bitonic sort of one key per lane across the warp.
__device__ __forceinline__ uint64_t warp_sort(uint64_t x) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1)
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const uint64_t y = __shfl_xor_sync(0xffffffffu, x, stride);
            const bool up = (lane & size) == 0 || size == 32;
            const bool lower = (lane & stride) == 0;
            x = (lower == up) ? umin64(x, y) : umax64(x, y);
        }
    return x;
}

// A warp-wide sorted list: lane j holds the j-th best key seen (ascending, 32 entries of
// which the first k matter); thr = entry k-1, thr_s its score (-inf while thr is ~0).  Single passing keys are inserted with a
// ballot + shuffle-up; bursts (a fresh list, a better row) are sorted and merged bitonically.
struct WarpTopK {
    uint64_t v;
    uint64_t thr;
    float thr_s;
    int k;
    __device__ __forceinline__ void init(int k_) {
        v = ~0ull, thr = ~0ull, thr_s = -INFINITY, k = k_;
    }
    __device__ __forceinline__ void refresh() {
        thr = __shfl_sync(0xffffffffu, v, k - 1);
        thr_s = thr == ~0ull ? -INFINITY : unordered(~uint32_t(thr >> 32));
    }
    __device__ __forceinline__ void insert(uint64_t key) {  // warp-uniform key
        const int lane = threadIdx.x & 31;
        const uint64_t up = __shfl_up_sync(0xffffffffu, v, 1);
        const int pos = __popc(__ballot_sync(0xffffffffu, v < key));
        v = lane < pos ? v : (lane == pos ? key : up);
    }
    __device__ __forceinline__ void merge_sorted(uint64_t c) {  // c: ascending across lanes
        const int lane = threadIdx.x & 31;
        uint64_t m = umin64(v, __shfl_sync(0xffffffffu, c, 31 - lane));  // bitonic: 32 smallest
#pragma unroll
        for (int stride = 16; stride > 0; stride >>= 1) {
            const uint64_t y = __shfl_xor_sync(0xffffffffu, m, stride);
            m = (lane & stride) == 0 ? umin64(m, y) : umax64(m, y);
        }
        v = m;
    }
    // Offer one key per lane.
    __device__ __forceinline__ void offer(uint64_t key) {
        unsigned m = __ballot_sync(0xffffffffu, key < thr);
        if (__popc(m) > 4) {
            merge_sorted(warp_sort(key < thr ? key : ~0ull));
            refresh();
            return;
        }
        while (m) {
            const int src = __ffs(m) - 1;
            m &= m - 1;
            const uint64_t kk = __shfl_sync(0xffffffffu, key, src);
            if (kk < thr) {
                insert(kk);
                refresh();
            }
        }
    }
    // Offer candidate (score s = base + v, token t, parent i) per lane.  The float pre-filter
    // s >= thr_s is necessary for key < thr, so the common case is one compare + ballot;
    // the key (and the reference's finiteness test on v) only for the few that pass.
    __device__ __forceinline__ void offer_score(float s, float v, int t, int i) {
        if (__ballot_sync(0xffffffffu, s >= thr_s) == 0u) return;
        offer(s >= thr_s && isfinite(v) ? rank_key(s, t, i) : ~0ull);
    }
};

// Merge the block's warp lists into warp 0's (lists staged in smem [kBeamWarps][32]).
__device__ __forceinline__ void block_merge(WarpTopK& wl, uint64_t* stage) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    stage[warp * 32 + lane] = lane < wl.k ? wl.v : ~0ull;
    __syncthreads();
    if (warp == 0)
        for (int w = 1; w < kBeamWarps; ++w) wl.offer(stage[w * 32 + lane]);
}

// Phase 1: CTA (split, b) scans its share of input b's first `roots` rows and writes its k
// best keys to part[(b*splits+split)*k].  Each row is read as float4 from its first 16-B
// aligned column (the <= 3 head / tail columns go through warp 0 of the first / last
// split); split s takes vector indices [s*cv, (s+1)*cv).  The filter is one max over the
// float4 against the row-adjusted threshold (loosened by a few ulps, as s = base + v rounds)
// per 4 columns; candidates that pass take the exact path (offer_score).  Loads are
// software-pipelined one batch ahead.
__global__ void __launch_bounds__(kBeamThreads) beam_scan_kernel(const float* __restrict__ lprobs,
                                                                 const float* __restrict__ live_lp, int lanes, int roots,
                                                                 int V, int k, int cv, uint64_t* __restrict__ part,
                                                                 const float* __restrict__ penalty) {
    __shared__ uint64_t stage[kBeamWarps * 32];
    const int split = blockIdx.x, b = blockIdx.y, splits = gridDim.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    WarpTopK wl;
    wl.init(k);
    constexpr int kStride = kBeamThreads * kUnroll;  // vector indices per CTA batch
    const int q0 = split * cv + warp * 32 + lane;
    const int per_row = cv - warp * 32 > 0 ? (cv - warp * 32 + kStride - 1) / kStride : 0;
    const int iters = per_row * roots;
    auto row_of = [&](int i) { return lprobs + (int64_t(b) * lanes + i) * V; };
    auto head_of = [&](const float* row) { return min(V, int((4 - ((reinterpret_cast<uintptr_t>(row) >> 2) & 3)) & 3)); };
    auto load = [&](int j, float4 (&v)[kUnroll]) {
        const int i = j / per_row;
        const float* row = row_of(i < roots ? i : 0);
        const int head = head_of(row);
        const int nvec = (V - head) >> 2;
        const float4* vrow = reinterpret_cast<const float4*>(row + head);
        const int q = q0 + (j - i * per_row) * kStride;
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const int qq = q + u * kBeamThreads;
            v[u] = (j < iters && qq < nvec && qq < (split + 1) * cv) ? __ldcs(vrow + qq)
                                                                     : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
        }
    };
    // scalar head / tail columns of every row
    if (warp == 0 && (split == 0 || split == splits - 1)) {
        for (int i = 0; i < roots; ++i) {
            const float* row = row_of(i);
            const int head = head_of(row);
            const int tail0 = head + (((V - head) >> 2) << 2);
            const float base = live_lp[int64_t(b) * lanes + i];
            int t = -1;
            if (split == 0 && lane < head && lane < V) t = lane;
            if (split == splits - 1 && lane >= 4 && lane - 4 < V - tail0 && tail0 + lane - 4 >= head) t = tail0 + lane - 4;
            const float v = t >= 0 ? row[t] : -INFINITY;
            const float pv = penalty != nullptr && t >= 0 ? penalty[int64_t(b) * V + t] : 0.f;
            wl.offer_score(base + (v - pv), v, t < 0 ? 0 : t, i);
        }
    }
    auto process = [&](int j, const float4 (&cur)[kUnroll]) {
        const int i = j / per_row;
        const float base = live_lp[int64_t(b) * lanes + i];
        const int head = head_of(row_of(i));
        const int q = q0 + (j - i * per_row) * kStride;
        // Pre-filter all batches first; the rare exact path is one code copy (a fully
        // inlined exact path per batch blows the kernel past the instruction cache).
        float vthr = (wl.thr_s - base) - (fabsf(wl.thr_s) + fabsf(base)) * 2.4e-7f;
        if (vthr != vthr) vthr = -INFINITY;
        unsigned pend = 0;
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const float4 x = cur[u];
            const float mx = fmaxf(fmaxf(x.x, x.y), fmaxf(x.z, x.w));
            if (__ballot_sync(0xffffffffu, mx >= vthr)) pend |= 1u << u;
        }
        while (pend) {
            const int u = __ffs(pend) - 1;
            pend &= pend - 1;
            float4 x = cur[0];
#pragma unroll
            for (int uu = 1; uu < kUnroll; ++uu)
                if (uu == u) x = cur[uu];
            const int t = head + 4 * (q + u * kBeamThreads);
#pragma unroll 1
            for (int e = 0; e < 4; ++e) {
                const float v = e == 0 ? x.x : (e == 1 ? x.y : (e == 2 ? x.z : x.w));
                const float pv = penalty != nullptr ? penalty[int64_t(b) * V + t + e] : 0.f;
                wl.offer_score(base + (v - pv), v, t + e, i);
            }
        }
    };
    // two register buffers, alternated without copies: one batch lands while the other is
    // filtered
    float4 bufA[kUnroll], bufB[kUnroll];
    if (iters > 0) load(0, bufA);
    for (int j = 0; j < iters; j += 2) {
        load(j + 1, bufB);
        process(j, bufA);
        if (j + 1 >= iters) break;
        load(j + 2, bufA);
        process(j + 1, bufB);
    }
    block_merge(wl, stage);
    if (threadIdx.x < k) part[(int64_t(b) * splits + split) * k + threadIdx.x] = wl.v;
}

// Phase 2: one warp per input merges its splits x k keys and decodes them.
__global__ void __launch_bounds__(32) beam_merge_kernel(const uint64_t* __restrict__ part, int splits, int k,
                                                        int* __restrict__ parent, int* __restrict__ token,
                                                        float* __restrict__ lp_sum) {
    const int b = blockIdx.x, lane = threadIdx.x;
    WarpTopK wl;
    wl.init(k);
    const uint64_t* in = part + int64_t(b) * splits * k;
    for (int c = lane; c < ((splits * k + 31) & ~31); c += 32) wl.offer(c < splits * k ? in[c] : ~0ull);
    if (lane < k) {
        const int64_t o = int64_t(b) * k + lane;
        const uint64_t key = wl.v;
        if (key == ~0ull) {
            parent[o] = -1, token[o] = -1, lp_sum[o] = -INFINITY;
        } else {
            parent[o] = int(key & 0xffu);
            token[o] = int((key >> 8) & 0xffffffu);
            lp_sum[o] = unordered(~uint32_t(key >> 32));
        }
    }
}

}  // namespace

// Column splits per input: about 2 CTAs per SM in total (ELATTN_BEAM_CTAS_PER_SM), chunks of >= 2048
// columns (ELATTN_BEAM_SPLITS overrides, for sweeps).
int beam_splits(int B, int V) {
    static const int forced = [] {
        const char* e = std::getenv("ELATTN_BEAM_SPLITS");
        return e ? std::atoi(e) : 0;
    }();
    const int cap = (V + 2047) / 2048;
    if (forced > 0) return forced < cap ? forced : (cap < 1 ? 1 : cap);
    static const int per_sm = [] {
        const char* e = std::getenv("ELATTN_BEAM_CTAS_PER_SM");
        return e ? std::atoi(e) : 2;
    }();
    const int want = (148 * per_sm + B - 1) / B;
    return want < 1 ? 1 : (want > cap ? (cap < 1 ? 1 : cap) : want);
}

void launch_beam_topk(const float* lprobs, const float* live_lp, const float* penalty, int B, int lanes, int roots,
                      int V, int k,
                      uint64_t* part, int splits, int* parent, int* token, float* lp_sum,
                      cudaStream_t st) {
    ELA_REQUIRE(k >= 1 && k <= kMaxK, ELATTN_ERR_UNSUPPORTED, "beam_candidates: k must be in [1, 32]");
    ELA_REQUIRE(lanes >= 1 && lanes <= 256 && roots >= 1 && roots <= lanes, ELATTN_ERR_SHAPE,
                "beam_candidates: 1 <= roots <= lanes <= 256");
    ELA_REQUIRE(V >= 1 && V < (1 << 24), ELATTN_ERR_SHAPE, "beam_candidates: vocabulary must be < 2^24");
    const int cv = ((V + 3) / 4 + splits - 1) / splits;
    beam_scan_kernel<<<dim3(splits, B), kBeamThreads, 0, st>>>(lprobs, live_lp, lanes, roots, V, k, cv, part,
                                                               penalty);
    ELA_CHECK_LAUNCH();
    beam_merge_kernel<<<B, 32, 0, st>>>(part, splits, k, parent, token, lp_sum);
    ELA_CHECK_LAUNCH();
}

}  // namespace elattn_gpu
