// el_decode_tc.cu — the fused EL-attention decode kernel for sm_100a (bf16).
//
// Computes, for every input b and each of its `rows` (= beams x heads) EL-Q rows,
//     C = softmax(q' . H_b^T / sqrt(d_k)) . H_b                      (fp32 accumulate)
// i.e. the core of el_attention_folded (attention.hpp:272-280), reading H_b from
// HBM exactly once and using every staged tile as BOTH key and value.
//
// Work split — thread-block CLUSTERS of 2 CTAs, split along d_m; persistent:
//   each cluster walks a list of SEGMENTS (whole inputs c, c + #clusters, ..., or — when
//   the last round is short — a stream-K chunk of the B*T tiles, whose partial inputs
//   are combined by el_decode_merge_kernel) as one continuous pipeline: a cluster-global
//   tile counter drives every ring / buffer phase across segments, so the next segment's
//   q' and H tiles stream in while the previous one drains.  Inputs with more than 64
//   query rows run as rows/64 virtual inputs sharing H.
//   CTA r owns d_m columns [r*d_m/2, (r+1)*d_m/2).  Its EL-Q half q'_r (64 x d_m/2)
//   is held half in TMEM (as the A operand of the score MMA) and half in smem; H_b
//   streams through a TMA ring in tiles of 32 rows x d_m/2 (SWIZZLE_128B, 128-column
//   "units" of 8 KB).  Per tile:
//     S_r   = q'_r . H_tile,r^T         tcgen05.mma M=64 N=32, K = d_m/2   (TMEM)
//     S     = S_0 + S_1                  partial scores swapped through DSMEM
//                                        (st.async + mbarrier complete_tx)
//     P     = exp2(S*scale*log2e - m)    online softmax, lazy rescale (FA4-style,
//                                        threshold 2^8)
//     O_r^T += H_tile,r^T . P^T          tcgen05.mma M=128 (d_m) N=64 (queries),
//                                        A = the SAME smem tile read MN-major
//   O_r (d_m/2 x 64 fp32) lives in TMEM for the whole input; the epilogue divides
//   by the softmax sums and writes C rows b*rows + q, columns of this CTA's half
//   (tcgen05.ld -> stmatrix.trans stage -> TMA store), optionally with the rows'
//   softmax statistics {m, l} (mixed self-attention).
// Both CTAs see bit-identical S (fp32 add commutes), so their softmax decisions agree.
//
// One thread can issue only ~1 tcgen05.mma per 56 cycles (tools/probes/
// mma_rate_probe.cu) and a score tile is 32 small MMAs, so three warps issue MMAs:
// S for even tiles, S for odd tiles, and O.  S runs up to 4 tiles ahead of O.
//
// Roles (384 threads, 12 warps):
//   warp 0      TMA producer (q' smem half, H ring)
//   warp 1      S issuer, even tiles (+ TMEM allocation owner)
//   warps 2..5  softmax / rescale / epilogue (TMEM lane quadrant = warp % 4)
//   warps 6..9  score exchange with the peer CTA, q' -> TMEM fill
//   warp 10     O issuer
//   warp 11     S issuer, odd tiles
#include "common.cuh"
#include "kernels.h"
#include "ptx_sm100.cuh"
#include "timeline.cuh"
#include "tmap.h"

#include <algorithm>
#include <cstdlib>

namespace elattn_gpu {

unsigned long long* g_decode_trace = nullptr;  // testing hook (elattn_gpu_testing_set_decode_trace)
int g_decode_sched_override = 0;  // testing hook: 0 auto, 1 stream-K, 2 whole inputs, 3 tail-split

namespace {

constexpr int kRowsQ = 64;         // EL-Q rows per input (padded)
constexpr int kNT = 32;            // H rows per tile
constexpr int kUnitBytes = 8192;   // 32 rows x 128 d_m x bf16
constexpr int kChunkBytes = 4096;  // 32 rows x 64 d_m
constexpr int kThreads = 384;
constexpr int kSBuf = 4;  // S accumulators in TMEM
constexpr int kEpiWarpBytes = 4096;  // per-warp epilogue stage (64 q x 32 d bf16), aliases P
// partial record of a split input, per (slot, CTA rank): m[64], l[64] (fp32), then per O
// unit the 128 softmax threads' 64 unnormalised fragment values in bf16 (4 values = 8 bytes
// per slot, interleaved by thread so every store / load is coalesced)
constexpr int kPartFloatsHdr = 128;
constexpr int kPartFloatsUnit = 128 * 32;  // 32-bit words: 64 bf16 values per softmax thread
constexpr int kQPrefetchTiles = 8;  // next segment's q' is prefetched into L2 this many tiles ahead
constexpr float kRescaleThreshold = 8.0f;
constexpr int kLptMaxTiles = 64;   // ragged longest-first: tile-count buckets (n_stride <= 2048)
constexpr int kLptMaxList = 32;    // ragged longest-first: inputs per cluster
// ragged schedules (static shared memory: the Sched objects of the six roles carry no
// pointer to them): stream-K chunk {g0, g_end, b0, prefix} / longest-first list length,
// the longest-first input list and the tile-count histogram
__shared__ int s_rsched[4];
__shared__ uint16_t s_lpt_list[kLptMaxList];
__shared__ int s_lpt_hist[kLptMaxTiles + 1];  // log2 domain: rescale only when max grows by > 2^8

// Tuning knobs (runtime so they can be swept):
//   s_ahead  — how many tiles S may run ahead of O (<= kSBuf);
//   l2_ahead — how many tiles ahead of the smem ring H is prefetched into L2 (0 = off).
struct DecodeTuning {
    int s_ahead = 4;
    int l2_ahead = 0;
    int skip_c_store = 0;  // TRACE builds only: drop the epilogue's global stores (timing experiments)
};
DecodeTuning g_tuning;

// TMEM columns (512): O^T [0, 64*UNITS) | S buffers [64*UNITS, +128) | q' units held in
// TMEM as the M=64 A operand [.., 512).  q' units that do not fit stay in smem.
template <int UNITS>
struct DecLayout {
    static constexpr int kTmemO = 0;
    static constexpr int kTmemS = 64 * UNITS;
    static constexpr int kTmemQ = kTmemS + 32 * kSBuf;
    static constexpr int kQTmemUnits = (512 - kTmemQ) / 64 < UNITS ? (512 - kTmemQ) / 64 : UNITS;
    static constexpr int kQSmemUnits = UNITS - kQTmemUnits;
    // shared memory
    static constexpr uint32_t kQBytes = kQSmemUnits * 2 * 8192;  // 64 rows x 128 d_m per unit
    static constexpr uint32_t kFixed =
        kQBytes + 2 * 8192 /*P*/ + 2 * 8192 /*recv*/ + 2 * 64 * 4 + 64 * 4 + 1024;
    static constexpr int kRingMax = 24;
    static constexpr int kRingFit = int((232448u - kFixed - 512u) / 8192u);
    static constexpr int kRing = kRingFit < kRingMax ? kRingFit : kRingMax;  // 8 KB units in the H ring
    static constexpr uint32_t kRingOff = kQBytes;
    static constexpr uint32_t kPOff = kRingOff + kRing * kUnitBytes;  // 2 x (64 rows x 128 B)
    static constexpr uint32_t kRecvOff = kPOff + 2 * 8192;            // 2 x (64 x 32 fp32)
    static constexpr uint32_t kAlphaOff = kRecvOff + 2 * 8192;        // 2 x 64 fp32
    static constexpr uint32_t kLOff = kAlphaOff + 2 * 64 * 4;         // 64 fp32
    static constexpr uint32_t kBarOff = kLOff + 64 * 4;
    static constexpr int kNumBars = 2 * kRing + 24;
    // + tmem slot; the ragged schedules' state is static shared memory (s_rsched, s_lpt_*)
    static constexpr uint32_t kStaticSmem = 16 + kLptMaxList * 2 + (kLptMaxTiles + 1) * 4 + 64;
    static constexpr uint32_t kTotal = kBarOff + kNumBars * 8 + 16 + 1024;
    static_assert(kTotal + kStaticSmem <= 232448, "shared memory budget");
    static_assert(kQTmemUnits >= 1, "at least one q' unit in TMEM");
    static_assert(4 * kEpiWarpBytes <= 2 * 8192, "epilogue stages alias the two P buffers");
};

__device__ __forceinline__ uint32_t softmax_bar_or(uint32_t pred) {
    uint32_t out;
    asm volatile(
        "{\n"
        ".reg .pred p, q;\n"
        "setp.ne.u32 q, %1, 0;\n"
        "bar.red.or.pred p, 1, 128, q;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(out)
        : "r"(pred)
        : "memory");
    return out;
}
__device__ __forceinline__ void softmax_bar_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// byte offset of (buffer, quadrant, k, lane) in the partial-score exchange buffer:
// float4-interleaved so both the remote writes and the local reads are conflict-free
__device__ __forceinline__ uint32_t recv_slot(int sb, uint32_t qd, int k, uint32_t lane) {
    return uint32_t((((sb * 4 + int(qd)) * 4 + k) * 32 + int(lane)) * 16);
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
}

// b is a VIRTUAL input: inputs with more than 64 query rows (beam > 4 at 16 heads) are
// processed as ceil(rows / 64) virtual inputs of up to 64 rows that share H_{b / vchunks}:
// virtual input b covers query rows [vrow0, vrow0 + vnrows) of the q' / C matrices.
__device__ __forceinline__ int vrow0(int b, int rows, int vchunks) {
    return (b / vchunks) * rows + (b % vchunks) * kRowsQ;
}
__device__ __forceinline__ int vnrows(int b, int rows, int vchunks) {
    return min(kRowsQ, rows - (b % vchunks) * kRowsQ);
}
__device__ __forceinline__ int tiles_of(const int* npi, int b, int n_stride, int vchunks) {
    const int n_b = npi ? npi[b / vchunks] : n_stride;
    return (n_b >= 1 && n_b <= n_stride) ? (n_b + kNT - 1) / kNT : 0;
}

// Work schedule of one cluster.  STREAM-K (uniform context length, T tiles per input) —
// the B*T tiles are cut into contiguous chunks of W tiles, one per cluster, so every
// cluster streams the same amount of H whatever B is (no wave tail, and small batches
// still use every SM).  An input cut by a chunk boundary is processed as SEGMENTS by
// consecutive clusters; each writes a partial record (unnormalised O, running max m, sum
// l) and el_decode_merge_kernel combines them in cluster order (deterministic).
// RAGGED STREAM-K (n_per_input given, moderate B): the same cut over the sum of the
// inputs' tile counts; every CTA finds its chunk start with a warp scan over n_per_input
// (the prefix is not known on the host) and the merge kernel repeats the scan.
// Otherwise (full last round, or many ragged inputs): whole inputs, cluster c takes c,
// c+ncl, ...
// RAGGED LONGEST-FIRST (default with n_per_input, no splitting): every CTA counting-sorts
// the inputs by tile count (descending, stable) in its prologue and takes sorted positions
// in boustrophedon order (round r: clusters 0..ncl-1, then ncl-1..0), the classic
// longest-processing-time-first approximation — whole inputs, no partial records.
struct SplitArgs {
    int T;           // tiles per input (uniform mode), 0 = ragged whole inputs (strided), -1 = ragged
                     // stream-K, -2 = ragged longest-first (list per cluster)
    int W;           // tiles per cluster chunk (uniform stream-K); -P: TAIL-SPLIT (see Sched);
                     // ragged stream-K: the minimum chunk (the chunk is max(W, ceil(tiles / ncl)))
    float* part;     // partial records [2 * ncl slots][2 ranks][kPartFloats]
    int vchunks;     // virtual inputs per real input (query rows / 64 when rows > 64)
    uint64_t h_pol;  // L2 policy of the H stream (evict-last when H fits in L2: the layers re-read it)
    int h_pre;       // H static across the stream's kernels (decoder step): tiles of the first segment
                     // loaded BEFORE the programmatic-dependent-launch wait (0 = after it)
    const int* h_index;  // MASK builds: input b reads H[h_index[b]] (slot-indexed lane caches; null = H[b])
};
// RAGGED: the ragged schedules (T < 0) are compiled only into the MASK instantiations (the
// ones launched with n_per_input); the production kernel keeps its schedule state minimal.
template <bool RAGGED>
struct Sched {
    int T, W, B, ncl, n_stride, vchunks;
    const int* npi;
    int g, g_end, b;
    bool first;
    // rs: ragged stream-K chunk of this cluster {g0, g_end, b0, prefix(b0)} (computed once per CTA)
    __device__ Sched(const SplitArgs& sa, int cl, int ncl_, int B_, int n_stride_, const int* npi_, const int* rs)
        : T(sa.T), W(sa.W), B(B_), ncl(ncl_), n_stride(n_stride_), vchunks(sa.vchunks), npi(npi_), first(true) {
        if (T > 0) {
            g = cl * W;
            g_end = min(B * T, g + W);
            b = cl;
        } else if (RAGGED && T == -1) {
            g = rs[0], g_end = rs[1], b = rs[2];
            W = rs[3];  // ragged stream-K: W holds the prefix (first global tile) of input b
        } else if (RAGGED && T == -2) {
            g = 0, g_end = rs[0];  // ragged longest-first: position in / length of this cluster's list
            b = 0;
        } else {
            g = g_end = 0;
            b = cl;
        }
    }
    // next segment: input bb, tiles [j0, j1) of its Tb; kind -1 = whole input, 0 = first
    // segment of this cluster's chunk, 1 = last segment (partial-record slot 2*cl + kind)
    __device__ bool next(int& bb, int& j0, int& j1, int& Tb, int& kind) {
        if (T > 0 && W < 0) {
            // TAIL-SPLIT: the full rounds as whole inputs (b = cl, cl + ncl, ... < Bw), then
            // part c % P of leftover input Bw + c / P, c = cl = b - Bw (no extra state: the
            // decode is sensitive to register pressure)
            const int Bw = B - B % ncl;
            if (b < Bw) {
                bb = b, j0 = 0, j1 = T, Tb = T, kind = -1;
                b += ncl;
                return true;
            }
            if (!first) return false;
            first = false;
            const int P = -W, c = b - Bw;
            if (c >= (B - Bw) * P) return false;
            bb = Bw + c / P;
            j0 = (T * (c % P)) / P;
            j1 = (T * (c % P + 1)) / P;
            Tb = T, kind = 0;
            return j1 > j0;
        }
        if (RAGGED && T == -2) {
            while (g < g_end) {
                bb = s_lpt_list[g++];
                Tb = tiles_of(npi, bb, n_stride, vchunks);
                if (Tb == 0) continue;
                j0 = 0, j1 = Tb, kind = -1;
                return true;
            }
            return false;
        }
        if (RAGGED && T < 0) {
            if (g >= g_end) return false;
            int tb = tiles_of(npi, b, n_stride, vchunks);
            while (W + tb <= g) {  // advance to the input holding tile g (W = its prefix)
                W += tb;
                tb = tiles_of(npi, ++b, n_stride, vchunks);
            }
            bb = b, Tb = tb;
            j0 = g - W;
            j1 = min(tb, g_end - W);
            kind = (j0 == 0 && j1 == tb) ? -1 : (first ? 0 : 1);
            first = false;
            g = W + j1;
            return true;
        }
        if (T > 0) {
            if (g >= g_end) return false;
            bb = g / T;
            j0 = g - bb * T;
            j1 = min(T, j0 + (g_end - g));
            Tb = T;
            g += j1 - j0;
            kind = (j0 == 0 && j1 == T) ? -1 : (first ? 0 : 1);
            first = false;
            return true;
        }
        for (; b < B; b += ncl) {
            Tb = tiles_of(npi, b, n_stride, vchunks);
            if (Tb == 0) continue;
            bb = b;
            j0 = 0;
            j1 = Tb;
            kind = -1;
            b += ncl;
            return true;
        }
        return false;
    }
};

// Ragged stream-K bookkeeping (one warp, all lanes): total tiles of the B (virtual) inputs,
// the chunk W = max(W_min, ceil(total / ncl)), and the input holding global tile g with its
// prefix (first global tile).  Inputs with an out-of-contract length count 0 tiles.
struct RaggedPos {
    int total, W, b, prefix;
};
__device__ __forceinline__ RaggedPos ragged_locate(const int* npi, int B, int n_stride, int vchunks, int ncl,
                                                   int W_min, int chunk_index, int g_override) {
    const int lane = int(threadIdx.x & 31);
    int tot = 0;
    for (int i = lane; i < B; i += 32) tot += tiles_of(npi, i, n_stride, vchunks);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    RaggedPos r;
    r.total = tot;
    r.W = max(W_min, (tot + ncl - 1) / ncl);
    const int g = g_override >= 0 ? g_override : chunk_index * r.W;
    r.b = B, r.prefix = tot;
    int base = 0;
    for (int i0 = 0; i0 < B && g < tot; i0 += 32) {
        const int t = i0 + lane < B ? tiles_of(npi, i0 + lane, n_stride, vchunks) : 0;
        int incl = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const int excl = base + incl - t;
        const unsigned m = __ballot_sync(0xffffffffu, t > 0 && excl <= g && g < excl + t);
        if (m) {
            const int src = __ffs(m) - 1;
            r.b = i0 + src;
            r.prefix = __shfl_sync(0xffffffffu, excl, src);
            break;
        }
        base += __shfl_sync(0xffffffffu, incl, 31);
    }
    return r;
}

// R16: instantiation for inputs of at most 16 query rows (one beam x 16 heads) — the epilogue
// moves a quarter of the O tile; the general instantiation keeps its register budget.
template <int UNITS, bool TRACE, bool MASK, bool R16 = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    el_decode_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_h,
                        const __grid_constant__ CUtensorMap tm_c,
                        const __nv_bfloat16* __restrict__ qp_rows, const int* __restrict__ n_per_input, int B,
                        int rows, int n_stride, int d_m, float scale_log2, __nv_bfloat16* __restrict__ ctx,
                        unsigned long long* __restrict__ trace, DecodeTuning tune, SplitArgs sa,
                        float2* __restrict__ stats, int pdl) {
    using L = DecLayout<UNITS>;
    constexpr int kRing = L::kRing;
    // optional per-tile clock64 trace of the first cluster (testing hook); G = cluster tile index.
    // Compiled only into the TRACE (instrumented) instantiation, like the tuning knobs below:
    // their checks cost ~3% in the production kernel.
#define ELA_TRACE(ev, G)                                                                          \
    do {                                                                                          \
        if constexpr (TRACE)                                                                      \
            if (trace != nullptr && blockIdx.x < 2 && (G) < 64)                                   \
                trace[(blockIdx.x * 32 + (ev)) * 64 + (G)] = clock64();                           \
    } while (0)
    constexpr int kTmemCols = 512;
    constexpr uint32_t kTmemS = L::kTmemS;
    extern __shared__ uint8_t smem_raw[];
    // 1024-B alignment for SWIZZLE_128B, by offsetting the __shared__ array itself so
    // the compiler keeps the shared address space (LDS/STS, not generic LD/ST)
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sq = smem;
    uint8_t* ring = smem + L::kRingOff;
    uint8_t* sP = smem + L::kPOff;
    float* recv = reinterpret_cast<float*>(smem + L::kRecvOff);
    float* s_alpha = reinterpret_cast<float*>(smem + L::kAlphaOff);
    float* s_l = reinterpret_cast<float*>(smem + L::kLOff);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
    uint64_t* q_full = bars;            // q' smem half landed (per input)
    uint64_t* q_empty = bars + 1;       // both S issuers finished reading q' (per input)
    uint64_t* q_tmem_full = bars + 2;   // q' TMEM half written by the exchange warps (per input)
    uint64_t* o_full = bars + 3;        // last O MMA of an input complete
    uint64_t* o_free = bars + 4;        // epilogue has read O out of TMEM
    uint64_t* o_done0 = bars + 5;       // per even tile: O MMAs complete
    uint64_t* s_full = bars + 6;        // [4]
    uint64_t* s_empty = s_full + kSBuf;  // [4]
    uint64_t* p_full = s_empty + kSBuf;  // [2]
    uint64_t* p_empty = p_full + 2;      // [2]
    uint64_t* recv_full = p_empty + 2;   // [2]
    uint64_t* recv_free = recv_full + 2;  // [2] arrived by the PEER's softmax warps
    uint64_t* unit_full = recv_free + 2;  // [kRing]
    uint64_t* unit_empty = unit_full + kRing;
    uint64_t* o_done1 = unit_empty + kRing;  // per odd tile: O MMAs complete
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done1 + 1);
    int* rsched = s_rsched;
    uint16_t* lpt_list = s_lpt_list;
    int* lpt_hist = s_lpt_hist;

    const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
    const uint32_t rank = ptx::cluster_ctarank(), peer = rank ^ 1u;
    const int cl = int(blockIdx.x >> 1), ncl = int(gridDim.x >> 1);
    const int dm_half = d_m / 2, dm_off = int(rank) * dm_half;
    const int total_rows = (B / sa.vchunks) * rows;  // B counts virtual inputs, rows real rows per input

    ELA_TL_DECL;
    if (threadIdx.x == 0) ELA_TRACE(29, 0);  // kernel entry
    if constexpr (TRACE)  // every CTA: %globaltimer at entry and exit (after the 2 x 32 x 64 event block)
        if (trace != nullptr && threadIdx.x == 0) trace[4096 + 2 * blockIdx.x] = ptx::globaltimer();
    if (warp == 0) {
        if (ptx::elect_one()) {
            ptx::prefetch_tmap(&tm_q);
            ptx::prefetch_tmap(&tm_h);
            ptx::prefetch_tmap(&tm_c);
            ptx::mbar_init(q_full, 1);
            ptx::mbar_init(q_empty, 2);
            ptx::mbar_init(q_tmem_full, 4);
            ptx::mbar_init(o_full, 1);
            ptx::mbar_init(o_free, 4);
            ptx::mbar_init(o_done0, 1);
            ptx::mbar_init(o_done1, 1);
            for (int i = 0; i < kSBuf; ++i) {
                ptx::mbar_init(&s_full[i], 1);
                ptx::mbar_init(&s_empty[i], 5);  // 4 exchange warps + the O issuer (softmax relay)
            }
            for (int i = 0; i < 2; ++i) {
                ptx::mbar_init(&p_full[i], 4);
                ptx::mbar_init(&p_empty[i], 1);
                ptx::mbar_init(&recv_full[i], 1);
                ptx::mbar_init(&recv_free[i], 4);
            }
            for (int s = 0; s < kRing; ++s) {
                ptx::mbar_init(&unit_full[s], 1);
                ptx::mbar_init(&unit_empty[s], 1);
            }
            ptx::fence_mbar_init();
            // expected bytes of the peer's partial scores for tiles 0 and 1; later
            // tiles are posted by the softmax warps once the previous phase is consumed
            ptx::mbar_arrive_expect_tx(&recv_full[0], kRowsQ * kNT * 4);
            ptx::mbar_arrive_expect_tx(&recv_full[1], kRowsQ * kNT * 4);
        }
        __syncwarp();
    } else if (warp == 1) {
        ptx::tmem_alloc<kTmemCols>(tmem_slot);
    }
    ptx::tc_fence_before();
    ptx::cluster_sync();  // peer barriers initialised before any st.async / remote arrive targets them
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    int n_pre = 0;  // tiles of the first segment already in flight (issued before the PDL wait)
    if (pdl) {
        // prologue done (TMEM held): the next kernel may launch; wait for the previous one
        ptx::griddep_launch_dependents();
        if constexpr (!MASK) {
            // H does not depend on the preceding kernels (the decoder step reads the encoder
            // state it was created with): start filling the ring now, so the first tiles'
            // HBM latency overlaps the q' expansion's tail; q' itself follows after the wait
            n_pre = sa.h_pre;
            if (warp == 0 && n_pre > 0) {
                Sched<MASK> pk(sa, cl, ncl, B, n_stride, n_per_input, rsched);
                int b0, j0, j1, Tb0, k0;
                if (!pk.next(b0, j0, j1, Tb0, k0)) j1 = j0;
                n_pre = min(n_pre, j1 - j0);
                if (ptx::elect_one()) {
                    for (int jj = 0; jj < n_pre; ++jj)
                        for (int u = 0; u < UNITS; ++u) {
                            const int s = jj * UNITS + u;  // first lap of the ring: slots are free
                            uint8_t* dst = ring + s * kUnitBytes;
                            ptx::mbar_arrive_expect_tx(&unit_full[s], kUnitBytes);
                            const int col = dm_off + 128 * u;
                            ptx::tma_load_3d(dst, &tm_h, &unit_full[s], col, (j0 + jj) * kNT, b0 / sa.vchunks, sa.h_pol);
                            ptx::tma_load_3d(dst + kChunkBytes, &tm_h, &unit_full[s], col + 64, (j0 + jj) * kNT,
                                             b0 / sa.vchunks, sa.h_pol);
                        }
                }
                __syncwarp();
            }
        }
        ptx::griddep_wait();
        ELA_TL_WAIT();
    }
    if (threadIdx.x == 0) ELA_TRACE(30, 0);  // setup done (after the PDL wait)
    if (MASK && sa.T == -2) {  // ragged longest-first: this cluster's inputs (n_per_input is read after the
                       // PDL wait: a preceding kernel may have written it)
        if (warp == 0) {
            const uint32_t lt_mask = (1u << lane) - 1u;
            // tile counts of inputs 512 s + 32 k + lane, k < 16: one round of sixteen loads in
            // flight per lane covers B <= 512 (reused by both passes)
            auto load16 = [&](int g0, int (&tl)[16]) {
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const int i = g0 + 32 * k + int(lane);
                    tl[k] = i < B ? min(tiles_of(n_per_input, i, n_stride, sa.vchunks), kLptMaxTiles) : -1;
                }
            };
            for (int t = int(lane); t <= kLptMaxTiles; t += 32) lpt_hist[t] = 0;
            __syncwarp();
            int tl[16];
            load16(0, tl);
            for (int g0 = 0; g0 < B; g0 += 512) {  // histogram of tile counts
                if (g0 > 0) load16(g0, tl);
#pragma unroll
                for (int k = 0; k < 16; ++k) {  // one add per distinct count (equal lengths: one per k)
                    const uint32_t peers = __match_any_sync(0xffffffffu, tl[k]);
                    if (tl[k] >= 0 && (peers & lt_mask) == 0) lpt_hist[tl[k]] += __popc(peers);
                    __syncwarp();
                }
            }
            __syncwarp();
            if (lane == 0) {  // bucket starts, longest first (then by input index)
                int acc = 0;
                for (int t = kLptMaxTiles; t >= 0; --t) {
                    const int c = lpt_hist[t];
                    lpt_hist[t] = acc;
                    acc += c;
                }
            }
            __syncwarp();
            int mine = 0;
            for (int g0 = 0; g0 < B; g0 += 512) {  // sorted position of every input -> its cluster
                if (g0 > 0 || B > 512) load16(g0, tl);
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const int t = tl[k];
                    const uint32_t peers = __match_any_sync(0xffffffffu, t);
                    const int pos = t >= 0 ? lpt_hist[t] + __popc(peers & lt_mask) : 0;
                    __syncwarp();
                    if (t >= 0 && (peers & lt_mask) == 0) lpt_hist[t] += __popc(peers);
                    const int r = pos / ncl, kk = pos - r * ncl;
                    const bool me = t >= 0 && ((r & 1) ? ncl - 1 - kk : kk) == cl;
                    if (me) lpt_list[r] = uint16_t(g0 + 32 * k + int(lane));
                    mine += __popc(__ballot_sync(0xffffffffu, me));
                    __syncwarp();
                }
            }
            if (lane == 0) rsched[0] = mine;  // positions r = 0..mine-1 are all filled (one per round)
        }
        __syncthreads();
    } else if (MASK && sa.T == -1) {  // ragged stream-K: this cluster's chunk of the inputs' tiles
        if (warp == 0) {
            const RaggedPos r = ragged_locate(n_per_input, B, n_stride, sa.vchunks, ncl, sa.W, cl, -1);
            if (lane == 0) {
                rsched[0] = min(cl * r.W, r.total);
                rsched[1] = min(cl * r.W + r.W, r.total);
                rsched[2] = r.b;
                rsched[3] = r.prefix;
            }
        }
        __syncthreads();
    }

    if (warp == 0) {
        // ================= TMA producer =================
        if (ptx::elect_one()) {
            int G = 0, li = 0;
            Sched<MASK> sc(sa, cl, ncl, B, n_stride, n_per_input, rsched);
            int b, j0, j1, Tb, kind;
            while (sc.next(b, j0, j1, Tb, kind)) {
                const int T = j1 - j0;
                // H block of this input (slot-indexed caches: a lane's history lives in its slot)
                const int hb = (MASK && sa.h_index != nullptr) ? __ldg(sa.h_index + b / sa.vchunks) : b / sa.vchunks;
                int nb = -1;  // input of the next segment (its q' is prefetched into L2)
                {
                    Sched<MASK> pk = sc;
                    int a0, a1, a2, a3;
                    if (!pk.next(nb, a0, a1, a2, a3)) nb = -1;
                }
                for (int jj = 0; jj < T; ++jj) {
                    const int j = j0 + jj, Gt = G + jj;
                    if (TRACE && tune.l2_ahead > 0 && j + tune.l2_ahead < Tb)
                        for (int c = 0; c < 2 * UNITS; ++c)
                            ptx::tma_prefetch_3d(&tm_h, dm_off + 64 * c, (j + tune.l2_ahead) * kNT, hb);
                    for (int u = 0; u < UNITS; ++u) {
                        const int g = Gt * UNITS + u, s = g % kRing;
                        if (Gt < n_pre) break;  // issued before the PDL wait
                        if (u == 0) ELA_TRACE(0, Gt);
                        ptx::mbar_wait(&unit_empty[s], ((g / kRing) & 1) ^ 1);
                        if (u == 0) ELA_TRACE(1, Gt);
                        uint8_t* dst = ring + s * kUnitBytes;
                        ptx::mbar_arrive_expect_tx(&unit_full[s], kUnitBytes);
                        const int col = dm_off + 128 * u;
                        // sibling virtual inputs (same H_b, running on neighbouring clusters)
                        // re-read the tile from L2: keep it there
                        const uint64_t pol = sa.h_pol;
                        ptx::tma_load_3d(dst, &tm_h, &unit_full[s], col, j * kNT, hb, pol);
                        ptx::tma_load_3d(dst + kChunkBytes, &tm_h, &unit_full[s], col + 64, j * kNT, hb,
                                         pol);
                    }
                    if (jj == (T > kQPrefetchTiles ? T - kQPrefetchTiles : 0) && nb >= 0 && nb != b) {
                        // warm L2 with the NEXT segment's q' (this CTA's d_m half) a few tiles
                        // before the transition (earlier, the streaming H evicts it again)
                        for (int c = 0; c < 2 * UNITS; ++c)
                            ptx::tma_prefetch_2d(&tm_q, dm_off + 64 * c, vrow0(nb, rows, sa.vchunks));
                    }
                    if (jj == 0 && L::kQSmemUnits > 0) {
                        // this input's smem half of q', once the previous input's S no longer reads it
                        if (li > 0) ptx::mbar_wait(q_empty, (li - 1) & 1);
                        ELA_TRACE(22, li);
                        ptx::mbar_arrive_expect_tx(q_full, L::kQBytes);
                        for (int c = 0; c < 2 * L::kQSmemUnits; ++c)
                            ptx::tma_load_2d(sq + c * 8192, &tm_q, q_full, dm_off + 128 * L::kQTmemUnits + 64 * c,
                                             vrow0(b, rows, sa.vchunks), ptx::kEvictFirst);  // q' is dead after this load
                    }
                }
                G += T;
                ++li;
            }
        }
        __syncwarp();
    } else if (warp == 1 || warp == 11) {
        // ================= S issuers (warp 1: even tiles, warp 11: odd tiles) =================
        // The whole warp runs the loop (slot/phase arithmetic stays warp-uniform, on the
        // uniform datapath next to UTCHMMA); lane 0 issues and commits.
        constexpr uint32_t idS = ptx::idesc_bf16(64, kNT, 0, 0);  // S = q' . H^T
        const uint64_t dRing = ptx::sdesc_sw128(ptx::smem_u32(ring), 0, 1024);
        const uint64_t dQ = ptx::sdesc_sw128(ptx::smem_u32(sq), 0, 1024);
        const int parity_mine = warp == 1 ? 0 : 1;
        int G = 0, li = 0;
        Sched<MASK> sc(sa, cl, ncl, B, n_stride, n_per_input, rsched);
        int b, j0, j1, Tb, kind;
        while (sc.next(b, j0, j1, Tb, kind)) {
            const int T = j1 - j0;
            // the TMEM half of q' (filled from registers) is usually ready before the smem
            // half (a TMA load after the previous segment's scores drained): start with the
            // TMEM units and wait for the smem half only when the first smem unit is due
            bool q_smem_ready = L::kQSmemUnits == 0;
            ptx::mbar_wait(q_tmem_full, li & 1);
            if (warp == 1 && lane == 0) ELA_TRACE(16, li);
            for (int Gt = G + ((G & 1) != parity_mine ? 1 : 0); Gt < G + T; Gt += 2) {
                const int sb = Gt & (kSBuf - 1);
                const uint32_t d = tmem + kTmemS + sb * kNT;
                if (lane == 0) ELA_TRACE(2, Gt);
                // buffer Gt%4 is free once the exchange warps and (relayed by the O
                // issuer) the softmax have consumed S(Gt-4)
                ptx::mbar_wait(&s_empty[sb], ((Gt / kSBuf) & 1) ^ 1);
                if (TRACE && tune.s_ahead < kSBuf && Gt >= tune.s_ahead) {
                    const int jj = Gt - tune.s_ahead;  // bound the lookahead: O(Gt - s_ahead) issued
                    ptx::mbar_wait(&s_empty[jj & (kSBuf - 1)], (jj / kSBuf) & 1);
                }
#pragma unroll
                for (int u = 0; u < UNITS; ++u) {
                    const int g = Gt * UNITS + u, slot = g % kRing;
                    if (u == L::kQTmemUnits && !q_smem_ready) {
                        ptx::mbar_wait(q_full, li & 1);
                        q_smem_ready = true;
                    }
                    ptx::mbar_wait(&unit_full[slot], (g / kRing) & 1);
                    ptx::tc_fence_after();
                    const uint64_t dB = dRing + uint64_t((slot * kUnitBytes) >> 4);
                    if (lane == 0) {
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk) {
                            const int h = kk >> 2, k16 = kk & 3;
                            const uint64_t bd = dB + uint64_t((h * kChunkBytes + 32 * k16) >> 4);
                            const uint32_t acc = (u | kk) != 0 ? 1u : 0u;
                            if (u < L::kQTmemUnits) {  // A (q') from TMEM: no smem operand traffic
                                ptx::mma_bf16_tmem_a(d, tmem + L::kTmemQ + u * 64 + kk * 8, bd, idS, acc);
                            } else {
                                const uint64_t a =
                                    dQ + uint64_t(((2 * (u - L::kQTmemUnits) + h) * 8192 + 32 * k16) >> 4);
                                ptx::mma_bf16(d, a, bd, idS, acc);
                            }
                        }
                    }
                    __syncwarp();
                }
                if (lane == 0) {
                    ptx::mma_commit(&s_full[sb]);
                    ELA_TRACE(3, Gt);
                }
                __syncwarp();
            }
            // this issuer is done reading the input's q' (smem + TMEM) once its MMAs drain
            if (lane == 0) ptx::mma_commit(q_empty);
            __syncwarp();
            G += T;
            ++li;
        }
    } else if (warp == 10) {
        // ================= O issuer =================
        constexpr uint32_t idO = ptx::idesc_bf16(128, 64, 1, 0);  // O^T += H^T . P^T (A MN-major)
        const uint64_t dRingMN = ptx::sdesc_sw128(ptx::smem_u32(ring), kChunkBytes, 1024);
        const uint64_t dP = ptx::sdesc_sw128(ptx::smem_u32(sP), 0, 1024);
        int G = 0, li = 0;
        Sched<MASK> sc(sa, cl, ncl, B, n_stride, n_per_input, rsched);
        int b, j0, j1, Tb, kind;
        while (sc.next(b, j0, j1, Tb, kind)) {
            const int T = j1 - j0;
            for (int j = 0; j < T; ++j) {  // j: tile index within the segment
                const int Gt = G + j, pb = Gt & 1;
                if (lane == 0) ELA_TRACE(4, Gt);
                ptx::mbar_wait(&p_full[pb], (Gt >> 1) & 1);
                // the first O of an input overwrites the accumulator: the previous
                // input's epilogue must have read it out
                if (j == 0 && li > 0) ptx::mbar_wait(o_free, (li - 1) & 1);
                if (j == 0 && lane == 0) ELA_TRACE(20, li);
                if (lane == 0) ELA_TRACE(5, Gt);
                ptx::tc_fence_after();
                if (lane == 0) {
#pragma unroll
                    for (int m = 0; m < UNITS; ++m) {
                        const int slot = (Gt * UNITS + m) % kRing;
#pragma unroll
                        for (int kk = 0; kk < kNT / 16; ++kk) {
                            const uint64_t a = dRingMN + uint64_t((slot * kUnitBytes + kk * 2048) >> 4);
                            const uint64_t bd = dP + uint64_t((pb * 8192 + 32 * kk) >> 4);
                            ptx::mma_bf16(tmem + m * 64, a, bd, idO, (j > 0 || kk > 0) ? 1u : 0u);
                        }
                        ptx::mma_commit(&unit_empty[slot]);
                    }
                    ptx::mma_commit(&p_empty[pb]);
                    ptx::mma_commit(pb ? o_done1 : o_done0);
                    // P(Gt) observed => the softmax has consumed S(Gt): release its buffer
                    ptx::mbar_arrive(&s_empty[Gt & (kSBuf - 1)]);
                }
                __syncwarp();
            }
            if (lane == 0) ptx::mma_commit(o_full);
            __syncwarp();
            G += T;
            ++li;
        }
    } else if (warp >= 6) {
        // ================= score exchange + q' TMEM fill (warps 6..9) =================
        const uint32_t qd = warp & 3;
        const uint32_t t_lane = tmem + ((qd * 32) << 16);
        const uint32_t peer_recv_full0 = ptx::mapa(ptx::smem_u32(&recv_full[0]), peer);
        const uint32_t peer_recv0 = ptx::mapa(ptx::smem_u32(recv), peer);
        // q' units [0, kQTmemUnits) of this CTA's d_m half -> TMEM, M=64 A layout (row
        // 16*qd + r in lane 32*qd + r, bf16 pairs packed per column), written with
        // tcgen05.st.16x256b so all 32 lanes carry data: thread t holds rows 16qd + t/4
        // and +8, columns 8k + 2(t%4) + {0,1}.  The NEXT input's q' is loaded into
        // registers right after this input's fill, so at the input transition the fill is
        // only the TMEM store.  Rows past an input's `rows` come from the next input (or
        // zeros past the end), matching the 64-row TMA box of the smem half.
        constexpr int kQW = 32 * L::kQTmemUnits;
        uint32_t qv[kQW];
        int qv_b = -1;
        auto q_load = [&](int bb) {
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const int q = int(qd) * 16 + int(lane >> 2) + 8 * half;
                const int r0 = vrow0(bb, rows, sa.vchunks);
                const bool ok = r0 + q < total_rows;
                const uint2* src =
                    reinterpret_cast<const uint2*>(qp_rows + (int64_t(r0) + q) * d_m + dm_off) + (lane & 3);
#pragma unroll
                for (int u = 0; u < L::kQTmemUnits; ++u)
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const uint2 v = ok ? __ldg(src + 32 * u + 4 * k) : make_uint2(0, 0);
                        qv[32 * u + 4 * k + 2 * half] = v.x;
                        qv[32 * u + 4 * k + 2 * half + 1] = v.y;
                    }
            }
            qv_b = bb;
        };
        int G = 0, li = 0;
        Sched<MASK> sc(sa, cl, ncl, B, n_stride, n_per_input, rsched);
        int b, j0, j1, Tb, kind;
        while (sc.next(b, j0, j1, Tb, kind)) {
            const int T = j1 - j0;
            {
                if (qv_b != b) q_load(b);
                if (li > 0) ptx::mbar_wait(q_empty, (li - 1) & 1);  // previous input's S done
                if (warp == 6 && lane == 0) ELA_TRACE(17, li);
#pragma unroll
                for (int u = 0; u < L::kQTmemUnits; ++u)
                    ptx::tmem_st_16x256b_x8(t_lane + L::kTmemQ + 64 * u, &qv[32 * u]);
                ptx::tmem_st_wait();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(q_tmem_full);
                if (warp == 6 && lane == 0) ELA_TRACE(18, li);
                {
                    Sched<MASK> pk = sc;  // the next segment's q' is in flight while this one streams
                    int nb, a0, a1, a2, a3;
                    if (pk.next(nb, a0, a1, a2, a3) && nb != b) q_load(nb);
                }
            }
            for (int j = 0; j < T; ++j) {
                const int Gt = G + j, sb = Gt & 1, sbuf = Gt & (kSBuf - 1);
                if (warp == 6 && lane == 0) ELA_TRACE(6, Gt);
                ptx::mbar_wait(&s_full[sbuf], (Gt / kSBuf) & 1);
                if (warp == 6 && lane == 0) ELA_TRACE(7, Gt);
                ptx::tc_fence_after();
                uint32_t sr[16];
                ptx::tmem_ld_16x256b_x4(t_lane + kTmemS + sbuf * kNT, sr);
                ptx::tmem_ld_wait();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&s_empty[sbuf]);
                // the peer must have consumed its recv[sb] of tile Gt-2
                ptx::mbar_wait(&recv_free[sb], ((Gt >> 1) & 1) ^ 1);
                if (warp == 6 && lane == 0) ELA_TRACE(8, Gt);
                const uint32_t rbar = peer_recv_full0 + sb * 8;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    ptx::st_async_v4(peer_recv0 + recv_slot(sb, qd, k, lane), __uint_as_float(sr[4 * k]),
                                     __uint_as_float(sr[4 * k + 1]), __uint_as_float(sr[4 * k + 2]),
                                     __uint_as_float(sr[4 * k + 3]), rbar);
                if (warp == 6 && lane == 0) ELA_TRACE(9, Gt);
            }
            G += T;
            ++li;
        }
    } else {
        // ================= softmax / rescale / epilogue (warps 2..5) =================
        // Score fragments are read with tcgen05.ld.16x256b so all 32 lanes work on
        // the M=64 tile: thread t owns query rows ra = 16*qd + t/4 and rb = ra + 8,
        // columns 8k + 2(t%4) + {0,1}; row reductions run over the 4-thread quad.
        const uint32_t qd = warp & 3;  // TMEM lane quadrant of this warp
        const int ra = int(qd) * 16 + int(lane >> 2), rb = ra + 8;
        const int cpair = 2 * int(lane & 3);
        const uint32_t t_lane = tmem + ((qd * 32) << 16);
        const uint32_t recv_base = ptx::smem_u32(recv);
        const uint32_t peer_recv_free0 = ptx::mapa(ptx::smem_u32(&recv_free[0]), peer);
        const float neg_inf = -INFINITY;
        // total tiles of this cluster (to stop arming recv_full past the end)
        int G_total = 0;
        int b, j0, j1, Tb, kind;
        {
            Sched<MASK> pk(sa, cl, ncl, B, n_stride, n_per_input, rsched);
            while (pk.next(b, j0, j1, Tb, kind)) G_total += j1 - j0;
        }
        int G = 0, li = 0;
        Sched<MASK> sc(sa, cl, ncl, B, n_stride, n_per_input, rsched);
        while (sc.next(b, j0, j1, Tb, kind)) {
            const int T = j1 - j0;
            const int n_b = n_per_input ? n_per_input[b / sa.vchunks] : n_stride;
            // MASK: ragged lengths or n not a multiple of the tile (else no tile is partial)
            const bool zero_tail = MASK && (n_per_input != nullptr) && (Tb * kNT > n_b);
            float m_a = neg_inf, m_b = neg_inf, l_a = 0.f, l_b = 0.f;  // running max (raw units), sums
            for (int jj = 0; jj < T; ++jj) {
                const int j = j0 + jj;  // tile index within the input
                const int Gt = G + jj, sb = Gt & 1, sbuf = Gt & (kSBuf - 1);
                const uint32_t par = (Gt >> 1) & 1;
                if (warp == 2 && lane == 0) ELA_TRACE(10, Gt);
                ptx::mbar_wait(&s_full[sbuf], (Gt / kSBuf) & 1);
                ptx::tc_fence_after();
                uint32_t sr[16];
                ptx::tmem_ld_16x256b_x4(t_lane + kTmemS + sbuf * kNT, sr);
                ptx::mbar_wait(&recv_full[sb], par);
                if (warp == 2 && lane == 0) {
                    ELA_TRACE(11, Gt);
                    // this phase is consumed: arm the same buffer for tile Gt+2
                    if (Gt + 2 < G_total) ptx::mbar_arrive_expect_tx(&recv_full[sb], kRowsQ * kNT * 4);
                }
                ptx::tmem_ld_wait();
                const int nvalid = min(kNT, n_b - j * kNT);
                float s[16];  // raw scores S_0 + S_1 (scale folded into the exponent below)
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float4 v = ptx::lds_f4(recv_base + recv_slot(sb, qd, k, lane));
                    s[4 * k + 0] = __uint_as_float(sr[4 * k + 0]) + v.x;
                    s[4 * k + 1] = __uint_as_float(sr[4 * k + 1]) + v.y;
                    s[4 * k + 2] = __uint_as_float(sr[4 * k + 2]) + v.z;
                    s[4 * k + 3] = __uint_as_float(sr[4 * k + 3]) + v.w;
                }
                if (MASK && nvalid < kNT) {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
#pragma unroll
                        for (int i = 0; i < 4; ++i)
                            if (8 * k + cpair + (i & 1) >= nvalid) s[4 * k + i] = neg_inf;
                }
                float xa = fmaxf(fmaxf(s[0], s[1]), fmaxf(s[4], s[5]));
                float xb = fmaxf(fmaxf(s[2], s[3]), fmaxf(s[6], s[7]));
                xa = fmaxf(xa, fmaxf(fmaxf(s[8], s[9]), fmaxf(s[12], s[13])));
                xb = fmaxf(xb, fmaxf(fmaxf(s[10], s[11]), fmaxf(s[14], s[15])));
                xa = fmaxf(xa, __shfl_xor_sync(0xffffffffu, xa, 1));
                xb = fmaxf(xb, __shfl_xor_sync(0xffffffffu, xb, 1));
                xa = fmaxf(xa, __shfl_xor_sync(0xffffffffu, xa, 2));
                xb = fmaxf(xb, __shfl_xor_sync(0xffffffffu, xb, 2));
                // every value read from recv[sb] has reached a register (the shuffles above
                // consumed them), so the peer may refill the buffer — for tile Gt + 2; none
                // is sent past the schedule's end (so every remote operation into a CTA is
                // awaited by it, and the kernel can end on an execution-only cluster barrier)
                if (lane == 0 && Gt + 2 < G_total) ptx::mbar_arrive_remote(peer_recv_free0 + sb * 8);
                uint32_t need = 0;
                float alpha_a = 1.f, alpha_b = 1.f;
                // lazy rescale: the reference max only moves when the tile max exceeds it
                // by more than 2^8 in probability (identical decision in all 4 quad threads
                // and in both CTAs of the cluster)
                if ((xa - m_a) * scale_log2 > kRescaleThreshold) {
                    need = 1;
                    alpha_a = ptx::ex2((m_a - xa) * scale_log2);  // 0 on the first tile
                    l_a *= alpha_a;
                    m_a = xa;
                }
                if ((xb - m_b) * scale_log2 > kRescaleThreshold) {
                    need = 1;
                    alpha_b = ptx::ex2((m_b - xb) * scale_log2);
                    l_b *= alpha_b;
                    m_b = xb;
                }
                if ((lane & 3) == 0) {
                    s_alpha[sb * 64 + ra] = alpha_a;
                    s_alpha[sb * 64 + rb] = alpha_b;
                }
                const float ma_s = m_a * scale_log2, mb_s = m_b * scale_log2;
                uint32_t pa[4], pb[4];
                float sa = 0.f, sbs = 0.f;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float p0 = ptx::ex2(fmaf(s[4 * k], scale_log2, -ma_s));
                    const float p1 = ptx::ex2(fmaf(s[4 * k + 1], scale_log2, -ma_s));
                    const float p2 = ptx::ex2(fmaf(s[4 * k + 2], scale_log2, -mb_s));
                    const float p3 = ptx::ex2(fmaf(s[4 * k + 3], scale_log2, -mb_s));
                    sa += p0 + p1;
                    sbs += p2 + p3;
                    pa[k] = pack_bf16x2(p0, p1);
                    pb[k] = pack_bf16x2(p2, p3);
                }
                sa += __shfl_xor_sync(0xffffffffu, sa, 1);
                sbs += __shfl_xor_sync(0xffffffffu, sbs, 1);
                sa += __shfl_xor_sync(0xffffffffu, sa, 2);
                sbs += __shfl_xor_sync(0xffffffffu, sbs, 2);
                l_a += sa;
                l_b += sbs;
                if (warp == 2 && lane == 0) ELA_TRACE(12, Gt);
                // P[sb] is free once O(Gt-2) has consumed it
                ptx::mbar_wait(&p_empty[sb], par ^ 1);
                {
                    uint8_t* P = sP + sb * 8192;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        *reinterpret_cast<uint32_t*>(P + ra * 128 + ((k ^ (ra & 7)) << 4) + 2 * cpair) = pa[k];
                        *reinterpret_cast<uint32_t*>(P + rb * 128 + ((k ^ (rb & 7)) << 4) + 2 * cpair) = pb[k];
                    }
                }
                if (zero_tail && j == Tb - 1) {
                    // rows n_b.. of the last tile are in-bounds padding of H_b: zero them
                    // before they meet P = 0 in the MMA (0 * NaN would poison O).
                    const int r0 = n_b - j * kNT;
                    const int tid = int(threadIdx.x) - 64;
                    const int per_chunk = (kNT - r0) * 8;
                    for (int idx = tid; idx < UNITS * 2 * per_chunk; idx += 128) {
                        const int ch = idx / per_chunk, rem = idx % per_chunk;
                        const int r = r0 + rem / 8, c16 = rem % 8;
                        const int sl = (Gt * UNITS + ch / 2) % kRing;
                        *reinterpret_cast<uint4*>(ring + sl * kUnitBytes + (ch & 1) * kChunkBytes + r * 128 +
                                                  c16 * 16) = make_uint4(0, 0, 0, 0);
                    }
                }
                const uint32_t any = softmax_bar_or(need);
                if (any && jj > 0) {
                    // lazy rescale of the running O^T columns once O(Gt-1) is complete: O *= alpha.
                    // (o_done has one barrier per tile parity, so waits can be skipped: the
                    // barrier of Gt-1 cannot be a full phase ahead while P(Gt+1) is unposted)
                    ptx::mbar_wait((Gt - 1) & 1 ? o_done1 : o_done0, ((Gt - 1) >> 1) & 1);
                    ptx::tc_fence_after();
#pragma unroll 1
                    for (int m = 0; m < UNITS; ++m) {
#pragma unroll
                        for (int c0 = 0; c0 < 64; c0 += 16) {
                            uint32_t r[16];
                            ptx::tmem_ld16(t_lane + m * 64 + c0, r);
                            ptx::tmem_ld_wait();
#pragma unroll
                            for (int i = 0; i < 16; ++i)
                                r[i] = __float_as_uint(__uint_as_float(r[i]) * s_alpha[sb * 64 + c0 + i]);
                            ptx::tmem_st16(t_lane + m * 64 + c0, r);
                        }
                    }
                    ptx::tmem_st_wait();
                }
                ptx::fence_proxy_async_smem();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&p_full[sb]);
                if (warp == 2 && lane == 0) ELA_TRACE(13, Gt);
                if (warp == 2 && lane == 0) {
                    if (Gt == 0) ELA_TL_MARK(0);  // first P posted
                    ELA_TL_MARK(1);               // (last) P posted
                }
            }

            // ---- epilogue: C[b*rows + q][dm_off + d] = O^T[d][q] / l_q.
            // O^T comes out of TMEM with tcgen05.ld.16x256b (thread t: lanes d = t/4,
            // t/4+8, columns q = 2(t%4)+{0,1} per 8-column group), i.e. already in the
            // 8x8 bf16 fragment layout of stmatrix; stmatrix.trans turns each warp's
            // 32(d) x 64(q) slab into a [q][32 d] SWIZZLE_64B tile (4 KB, aliasing the P
            // buffers, which are free once O is complete), stored by one TMA store per
            // warp and unit.  No CTA-wide barrier per unit; the next input streams meanwhile.
            if (warp == 2 && lane == 0) ELA_TRACE(14, li);
            uint8_t* my_stage = sP + (warp - 2) * kEpiWarpBytes;
            // stmatrix row address of lane l: matrix j = l/8 (d 8j..8j+7), row i = l%8 (q = 8k+i);
            // SWIZZLE_64B: 16-byte chunk j of 64-byte row q sits at chunk j ^ ((q >> 1) & 3)
            const uint32_t stm_i = lane & 7, stm_j = lane >> 3;
            const uint32_t stm_base = ptx::smem_u32(my_stage) + stm_i * 64;
            const int tid = int(threadIdx.x) - 64;  // 0..127 over the softmax warps
            // unit m of the output: fp32 fragments lo/hi (lanes d 0..15 / 16..31 of the quadrant)
            // scaled by sc[] (per query column of this thread) -> bf16 -> stage -> TMA store
            auto emit_unit = [&](int m, const uint32_t(&lo)[32], const uint32_t(&hi)[32], const float(&sc)[16]) {
                if (warp == 2 && lane == 0) ELA_TRACE(24, li * 4 + m);
                __syncwarp();  // every lane has read the previous unit out of the stage
                if (warp == 2 && lane == 0) ELA_TRACE(25, li * 4 + m);
#pragma unroll
                for (int k = 0; k < 8; ++k) {  // query columns 8k..8k+7
                    uint32_t f[4];
                    const uint32_t* src[2] = {lo, hi};
#pragma unroll
                    for (int h2 = 0; h2 < 2; ++h2)
#pragma unroll
                        for (int half = 0; half < 2; ++half) {
                            const uint32_t* r = src[h2] + 4 * k + 2 * half;
                            f[2 * h2 + half] = pack_bf16x2(__uint_as_float(r[0]) * sc[2 * k],
                                                           __uint_as_float(r[1]) * sc[2 * k + 1]);
                        }
                    const uint32_t q = 8u * k + stm_i;
                    ptx::stmatrix_x4_trans(stm_base + k * 512 + ((stm_j ^ ((q >> 1) & 3u)) << 4), f[0], f[1], f[2],
                                           f[3]);
                }
                __syncwarp();
                if (warp == 2 && lane == 0) ELA_TRACE(26, li * 4 + m);
                // read the [64 q][32 d] stage back row-contiguous and store with st.global.v4:
                // each instruction writes 8 query rows x 64 bytes (no TMA-store round trip,
                // so the next unit can be staged at once and the next input's softmax is
                // not held up behind store-read latency)
                __nv_bfloat16* dst = ctx + int64_t(vrow0(b, rows, sa.vchunks)) * d_m + dm_off + m * 128 + int(qd) * 32;
                const int nr = vnrows(b, rows, sa.vchunks);
#pragma unroll
                for (int s8 = 0; s8 < 8; ++s8) {
                    const int q = s8 * 8 + int(lane >> 2), j = int(lane & 3);
                    const uint4 v = ptx::lds_u4(ptx::smem_u32(my_stage) + q * 64 + ((j ^ ((q >> 1) & 3)) << 4));
                    if (q < nr && !(TRACE && tune.skip_c_store))
                        *reinterpret_cast<uint4*>(dst + int64_t(q) * d_m + 8 * j) = v;
                }
                if (warp == 2 && lane == 0) ELA_TRACE(28, li * 4 + m);
            };
            // the same for inputs with at most 16 query rows (one beam x 16 heads: greedy
            // decoding, decoder-only lanes): a quarter of the TMEM loads, transposes and stores
            auto emit_unit16 = [&](int m, const uint32_t(&lo)[8], const uint32_t(&hi)[8], const float(&sc)[16]) {
                __syncwarp();
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    uint32_t f[4];
                    const uint32_t* src[2] = {lo, hi};
#pragma unroll
                    for (int h2 = 0; h2 < 2; ++h2)
#pragma unroll
                        for (int half = 0; half < 2; ++half) {
                            const uint32_t* r = src[h2] + 4 * k + 2 * half;
                            f[2 * h2 + half] = pack_bf16x2(__uint_as_float(r[0]) * sc[2 * k],
                                                           __uint_as_float(r[1]) * sc[2 * k + 1]);
                        }
                    const uint32_t q = 8u * k + stm_i;
                    ptx::stmatrix_x4_trans(stm_base + k * 512 + ((stm_j ^ ((q >> 1) & 3u)) << 4), f[0], f[1], f[2],
                                           f[3]);
                }
                __syncwarp();
                __nv_bfloat16* dst = ctx + int64_t(vrow0(b, rows, sa.vchunks)) * d_m + dm_off + m * 128 + int(qd) * 32;
                const int nr = vnrows(b, rows, sa.vchunks);
#pragma unroll
                for (int s8 = 0; s8 < 2; ++s8) {
                    const int q = s8 * 8 + int(lane >> 2), j = int(lane & 3);
                    const uint4 v = ptx::lds_u4(ptx::smem_u32(my_stage) + q * 64 + ((j ^ ((q >> 1) & 3)) << 4));
                    if (q < nr && !(TRACE && tune.skip_c_store))
                        *reinterpret_cast<uint4*>(dst + int64_t(q) * d_m + 8 * j) = v;
                }
            };
            if (kind < 0) {
                // whole input: normalise by 1/l and write
                if ((lane & 3) == 0) {
                    s_l[ra] = 1.f / l_a;
                    s_l[rb] = 1.f / l_b;
                    if (stats != nullptr && rank == 0) {  // softmax stats in log2 units (both CTAs agree)
                        const int r0 = vrow0(b, rows, sa.vchunks), nr = vnrows(b, rows, sa.vchunks);
                        if (ra < nr) stats[r0 + ra] = make_float2(m_a * scale_log2, l_a);
                        if (rb < nr) stats[r0 + rb] = make_float2(m_b * scale_log2, l_b);
                    }
                }
                softmax_bar_sync();
                float inv_l[16];  // 1/l for this thread's columns q = 8k + 2(t%4) + {0,1}
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const float2 v = *reinterpret_cast<const float2*>(s_l + 8 * k + cpair);
                    inv_l[2 * k] = v.x, inv_l[2 * k + 1] = v.y;
                }
                ptx::mbar_wait(o_full, li & 1);  // all O MMAs done: P buffers are free as stages
                ptx::tc_fence_after();
                if (warp == 2 && lane == 0) ELA_TRACE(19, li);
                // unit by unit: TMEM -> registers -> bf16 stage -> st.global (the stores do
                // not block, so no software pipelining is needed to hide them)
                if constexpr (R16) {
#pragma unroll 1
                    for (int m = 0; m < UNITS; ++m) {
                        uint32_t lo[8], hi[8];
                        ptx::tmem_ld_16x256b_x2(t_lane + m * 64, lo);
                        ptx::tmem_ld_16x256b_x2(t_lane + (16u << 16) + m * 64, hi);
                        ptx::tmem_ld_wait();
                        if (m == UNITS - 1) {  // O read out: the next segment may overwrite it
                            ptx::tc_fence_before();
                            __syncwarp();
                            if (lane == 0) ptx::mbar_arrive(o_free);
                        }
                        emit_unit16(m, lo, hi, inv_l);
                    }
                } else
#pragma unroll 1
                for (int m = 0; m < UNITS; ++m) {
                    uint32_t lo[32], hi[32];
                    ptx::tmem_ld_16x256b_x8(t_lane + m * 64, lo);
                    ptx::tmem_ld_16x256b_x8(t_lane + (16u << 16) + m * 64, hi);
                    ptx::tmem_ld_wait();
                    if (m == 0 && warp == 2 && lane == 0) ELA_TRACE(21, li);
                    if (m == UNITS - 1) {  // O read out: the next segment may overwrite it
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) ptx::mbar_arrive(o_free);
                    }
                    if (warp == 2 && lane == 0) ELA_TRACE(27, li * 4 + m);
                    emit_unit(m, lo, hi, inv_l);
                }
            } else {
                // segment of a split input: write its partial record (running max m and
                // sum l per query row, unnormalised O^T in this thread's fragment order);
                // el_decode_merge_kernel combines the records after this kernel
                constexpr int kPF = kPartFloatsHdr + UNITS * kPartFloatsUnit;
                float* rec = sa.part + (int64_t(2 * cl + kind) * 2 + rank) * kPF;
                if ((lane & 3) == 0) {
                    rec[ra] = m_a;
                    rec[rb] = m_b;
                    rec[64 + ra] = l_a;
                    rec[64 + rb] = l_b;
                }
                ptx::mbar_wait(o_full, li & 1);
                ptx::tc_fence_after();
#pragma unroll 1
                for (int m = 0; m < UNITS; ++m) {
                    uint32_t lo[32], hi[32];
                    ptx::tmem_ld_16x256b_x8(t_lane + m * 64, lo);
                    ptx::tmem_ld_16x256b_x8(t_lane + (16u << 16) + m * 64, hi);
                    ptx::tmem_ld_wait();
                    if (m == UNITS - 1) {
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) ptx::mbar_arrive(o_free);
                    }
                    uint2* body = reinterpret_cast<uint2*>(rec + kPartFloatsHdr + m * kPartFloatsUnit);
                    // evict-last: the merge kernel re-reads the records right after this
                    // kernel, and the H stream would otherwise push them out of L2
#pragma unroll
                    for (int i4 = 0; i4 < 8; ++i4) {
                        ptx::st_global_v2_hint(&body[(0 * 8 + i4) * 128 + tid],
                                               pack_bf16x2(__uint_as_float(lo[4 * i4]), __uint_as_float(lo[4 * i4 + 1])),
                                               pack_bf16x2(__uint_as_float(lo[4 * i4 + 2]), __uint_as_float(lo[4 * i4 + 3])),
                                               ptx::kEvictLast);
                        ptx::st_global_v2_hint(&body[(1 * 8 + i4) * 128 + tid],
                                               pack_bf16x2(__uint_as_float(hi[4 * i4]), __uint_as_float(hi[4 * i4 + 1])),
                                               pack_bf16x2(__uint_as_float(hi[4 * i4 + 2]), __uint_as_float(hi[4 * i4 + 3])),
                                               ptx::kEvictLast);
                    }
                }
            }
            if (warp == 2 && lane == 0) ELA_TRACE(23, li);
            // stages alias P: every warp has read its stage back before any warp writes P
            // of the next input
            softmax_bar_sync();
            if (warp == 2 && lane == 0) ELA_TRACE(15, li);
            if (warp == 2 && lane == 0) ELA_TL_MARK(2);  // (last) epilogue done
            G += T;
            ++li;
        }
        // inputs whose context length is out of contract: loud NaN rows
        for (int b = cl; b < B; b += ncl) {
            if (tiles_of(n_per_input, b, n_stride, sa.vchunks) != 0) continue;
            const int tid = int(threadIdx.x) - 64;
            const int r0 = vrow0(b, rows, sa.vchunks);
            for (int e = tid; e < vnrows(b, rows, sa.vchunks) * dm_half; e += 128)
                ctx[(int64_t(r0) + e / dm_half) * d_m + dm_off + e % dm_half] =
                    __float2bfloat16_rn(__int_as_float(0x7fc00000));
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) ELA_TRACE(31, 0);  // all roles done
    if constexpr (TRACE)
        if (trace != nullptr && threadIdx.x == 0) trace[4096 + 2 * blockIdx.x + 1] = ptx::globaltimer();
    // the peer stays alive until this CTA's DSMEM traffic into it has landed: every score
    // exchange completes on a recv_full the peer waited on, and no recv_free arrive is sent
    // past the schedule — execution-only barrier, the C / record stores drain at grid end
    ptx::cluster_sync_relaxed();
    ELA_TL_EXIT(kTlDecode);
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<kTmemCols>(tmem);
    }
#undef ELA_TRACE
}

int num_sms_decode() {
    static int n = [] {
        int dev = 0, v = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return n;
}

// Combines the partial records of every split input (stream-K) into C rows.
// CTA (chunk boundary k, rank r, unit m), 256 threads; only the CTA of the first boundary
// inside an input works.  Phase 1 (one thread per query row q): M = max_s m_s, per-segment
// weights w_s = 2^{(m_s - M) c} and 1/L, L = sum_s l_s w_s, into smem.  Phase 2: the unit's
// 2048 float4 fragments (written by the decode kernel's softmax thread t as lanes d rows
// 32 qd + t/4 + {0,8,16,24}, query columns 8k + 2(t%4) + {0,1}, qd = (t/32 + 2) & 3) are
// loaded for all segments at once, O = sum_s w_s O_s, scaled by 1/L, staged as a
// [64 q][128 d] bf16 tile and written with 16-byte stores.  Segment order is fixed
// (cluster order), so the result does not depend on timing.
constexpr int kMaxSegs = 8;
template <int UNITS>
__global__ void __launch_bounds__(256) el_decode_merge_kernel(const float* __restrict__ part, int T, int W, int ncl,
                                                              int rows, int vchunks, int d_m, float scale_log2,
                                                              __nv_bfloat16* __restrict__ ctx,
                                                              float2* __restrict__ stats, int Bw,
                                                              const int* __restrict__ npi, int B, int n_stride) {
    constexpr int kPF = kPartFloatsHdr + UNITS * kPartFloatsUnit;
    ELA_TL_DECL;
    // the next kernel (the V projection) may launch now and stage its weights; it waits for
    // this grid's completion before reading C
    ptx::griddep_launch_dependents();
    ptx::griddep_wait();  // launched with PDL after the decode: its records must be complete
    ELA_TL_WAIT();
    const int rank = int(blockIdx.y), m = int(blockIdx.z);
    int b, c_first, nseg;
    int64_t first_tile = 0;  // b's first tile in the cut (stream-K): decides each segment's record slot
    __shared__ int s_rag[4];  // ragged: b, prefix, tiles of b, chunk W (b < 0: no merge here)
    if (T < 0) {
        // ragged stream-K: the same scan as the decode kernel locates the input holding
        // boundary k*W, its prefix and tile count
        if (threadIdx.x < 32) {
            const int k = int(blockIdx.x) + 1;
            const RaggedPos r = ragged_locate(npi, B, n_stride, vchunks, ncl, W, k, -1);
            const int gk = k * r.W;
            const int tb = r.b < B ? tiles_of(npi, r.b, n_stride, vchunks) : 0;
            // merged at b's first interior boundary only
            const bool split = gk < r.total && gk != r.prefix && (k - 1) * r.W <= r.prefix;
            if (threadIdx.x == 0) {
                s_rag[0] = split ? r.b : -1;
                s_rag[1] = r.prefix;
                s_rag[2] = tb;
                s_rag[3] = r.W;
            }
        }
        __syncthreads();
        if (s_rag[0] < 0) return;
        b = s_rag[0];
        const int pb = s_rag[1];
        W = s_rag[3];
        first_tile = pb;
        c_first = pb / W;
        nseg = min(kMaxSegs, (pb + s_rag[2] - 1) / W - c_first + 1);
    } else if (W < 0) {  // tail-split: input Bw + x in P = -W parts on clusters P x .. P x + P - 1 (slot 0)
        b = Bw + int(blockIdx.x);
        c_first = int(blockIdx.x) * -W;
        nseg = -W;
    } else {
        const int k = int(blockIdx.x) + 1;
        const int64_t gk = int64_t(k) * W;
        b = int(gk / T);
        if (gk % T == 0 || int64_t(k - 1) * W > int64_t(b) * T) return;  // not a split, or not b's first boundary
        first_tile = int64_t(b) * T;
        c_first = int(first_tile / W);
        nseg = min(kMaxSegs, int((int64_t(b) * T + T - 1) / W) - c_first + 1);
    }
    __shared__ float s_w[kMaxSegs][64];
    __shared__ float s_inv[64];
    __shared__ __align__(16) __nv_bfloat16 tile[64][128 + 8];
    const int tid = int(threadIdx.x);
    auto rec_of = [&](int s) {  // record of segment s (cluster c_first + s; slot 0 unless b is its 2nd)
        const int c2 = c_first + s;
        const int kd = (W < 0 || int64_t(c2) * W >= first_tile) ? 0 : 1;
        return part + (int64_t(2 * c2 + kd) * 2 + rank) * kPF;
    };
    // fragment float4 e = (h * 8 + i4) * 128 + t of the unit; this thread takes e = tid + 256 j.
    // The fragments of the first kPre segments do not depend on the weights: all of their
    // loads are issued before phase 1, so the merge costs ~one L2 round trip, not nseg + 1
    constexpr int kPer = 2 * 8 * 128 / 256, kPre = 4;
    // the per-row maxima and sums first (phase 1 needs them before anything else), then
    // the fragments
    float ms[kMaxSegs], ls[kMaxSegs];
    if (tid < 64) {
#pragma unroll
        for (int s = 0; s < kMaxSegs; ++s)
            if (s < nseg) {
                const float* r = rec_of(s);
                ms[s] = __ldcg(r + tid);
                ls[s] = __ldcg(r + 64 + tid);
            }
    }
    uint2 vp[kPre][kPer];
#pragma unroll
    for (int s = 0; s < kPre; ++s)
        if (s < nseg) {
            const uint2* body = reinterpret_cast<const uint2*>(rec_of(s) + kPartFloatsHdr + m * kPartFloatsUnit);
#pragma unroll
            for (int j = 0; j < kPer; ++j) vp[s][j] = __ldcg(body + tid + 256 * j);
        }
    if (tid < 64) {
        float M = -INFINITY, L = 0.f;
#pragma unroll
        for (int s = 0; s < kMaxSegs; ++s)
            if (s < nseg) M = fmaxf(M, ms[s]);
#pragma unroll
        for (int s = 0; s < kMaxSegs; ++s)
            if (s < nseg) {
                const float w = ptx::ex2((ms[s] - M) * scale_log2);
                s_w[s][tid] = w;
                L += ls[s] * w;
            }
        s_inv[tid] = 1.f / L;
        if (stats != nullptr && rank == 0 && m == 0 && tid < vnrows(b, rows, vchunks))
            stats[vrow0(b, rows, vchunks) + tid] = make_float2(M * scale_log2, L);
        if (tid == 0) ELA_TL_MARK(0);  // segment weights ready
    }
    __syncthreads();
    float4 acc[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    auto accumulate = [&](int s, const uint2 (&v)[kPer]) {
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            const int e = tid + 256 * j, t = e & 127, i4 = (e >> 7) & 7;
            const int q0 = 8 * i4 + 2 * (t & 3);
            const float w0 = s_w[s][q0], w1 = s_w[s][q0 + 1];
            const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v[j].x));
            const float2 c = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v[j].y));
            acc[j].x += a.x * w0, acc[j].y += a.y * w1, acc[j].z += c.x * w0, acc[j].w += c.y * w1;
        }
    };
#pragma unroll
    for (int s = 0; s < kPre; ++s)
        if (s < nseg) accumulate(s, vp[s]);
    for (int s = kPre; s < nseg; ++s) {
        const uint2* body = reinterpret_cast<const uint2*>(rec_of(s) + kPartFloatsHdr + m * kPartFloatsUnit);
        uint2 v[kPer];
#pragma unroll
        for (int j = 0; j < kPer; ++j) v[j] = __ldcg(body + tid + 256 * j);
        accumulate(s, v);
    }
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        const int e = tid + 256 * j, t = e & 127, i4 = (e >> 7) & 7, h = e >> 10;
        const int qd = ((t >> 5) + 2) & 3, q0 = 8 * i4 + 2 * (t & 3);
        const int d0 = 32 * qd + 16 * h + ((t & 31) >> 2);  // regs x,y: d0; z,w: d0 + 8
        tile[q0][d0] = __float2bfloat16_rn(acc[j].x * s_inv[q0]);
        tile[q0 + 1][d0] = __float2bfloat16_rn(acc[j].y * s_inv[q0 + 1]);
        tile[q0][d0 + 8] = __float2bfloat16_rn(acc[j].z * s_inv[q0]);
        tile[q0 + 1][d0 + 8] = __float2bfloat16_rn(acc[j].w * s_inv[q0 + 1]);
    }
    __syncthreads();
    if (tid == 0) ELA_TL_MARK(1);  // merged tile staged
    const int dm_off = rank * (d_m / 2) + m * 128;
    const int r0 = vrow0(b, rows, vchunks);
    for (int e = tid; e < vnrows(b, rows, vchunks) * 16; e += 256) {
        const int q = e >> 4, v = e & 15;
        *reinterpret_cast<uint4*>(ctx + (int64_t(r0) + q) * d_m + dm_off + 8 * v) =
            *reinterpret_cast<const uint4*>(&tile[q][8 * v]);
    }
    if (tid == 0) ELA_TL_MARK(2);  // stores issued
    ELA_TL_EXIT(kTlMerge);
}

}  // namespace

ELA_TL_SETTER(tl_set_decode)

size_t el_decode_tc_scratch_bytes(int d_m) {
    // partial records of split inputs: 2 slots per cluster x 2 CTA ranks, at most one
    // cluster per pair of SMs (the schedule never uses more clusters than that)
    const size_t units = size_t(d_m / 256 < 1 ? 1 : d_m / 256);
    const size_t kPF = kPartFloatsHdr + units * kPartFloatsUnit;
    return size_t(2 * (num_sms_decode() / 2)) * 2 * kPF * sizeof(float);
}

namespace {

constexpr int kMinChunkTiles = 8;  // bounds the segments per input (merge cost) at small B
constexpr int kRaggedSkMaxInputs = 8;  // ragged stream-K up to 8 inputs per cluster (beyond: whole inputs)

template <int UNITS>
void launch_units(const void* qp, const void* H, const int* npi, int B, int rows, int n_stride, int d_m,
                  float scale_log2, void* ctx, cudaStream_t st, float2* stats, float* part, bool h_static,
                  const int* h_index, int h_slots) {
    // > 64 query rows per input: rows/64 virtual inputs of 64 rows each (q' and C rows are
    // contiguous per input, so virtual input v owns rows [64 v, 64 v + 64)); H_b is shared
    const int vchunks = rows > kRowsQ ? (rows + kRowsQ - 1) / kRowsQ : 1;
    const int B_h = B;
    B *= vchunks;  // virtual inputs; `rows` stays the real rows per input
    // q' viewed as [B*rows][d_m]; box 64 rows (rows < 64 pad with the next input's
    // rows or OOB zeros; only the first `rows` outputs are written).
    const uint64_t qdims[2] = {uint64_t(d_m), uint64_t(B_h) * rows};
    const uint64_t qstr[1] = {uint64_t(d_m) * 2};
    const uint32_t qbox[2] = {64, kRowsQ};
    CUtensorMap tq = make_tmap_bf16(qp, 2, qdims, qstr, qbox);
    const uint64_t hdims[3] = {uint64_t(d_m), uint64_t(n_stride), uint64_t(h_index ? h_slots : B_h)};
    const uint64_t hstr[2] = {uint64_t(d_m) * 2, uint64_t(n_stride) * d_m * 2};
    const uint32_t hbox[3] = {64, kNT, 1};
    CUtensorMap th = make_tmap_bf16(H, 3, hdims, hstr, hbox);
    // C viewed as [B*rows][d_m]; box = one input's rows x 32 columns (one softmax warp's
    // d slab of a unit), SWIZZLE_64B to match the stmatrix stage layout
    const uint64_t cdims[2] = {uint64_t(d_m), uint64_t(B_h) * rows};
    const uint32_t cbox[2] = {32, uint32_t(rows < kRowsQ ? rows : kRowsQ)};
    CUtensorMap tc = make_tmap_bf16(ctx, 2, cdims, qstr, cbox, 64);
    // instrumented instantiation (trace hook, lookahead knobs) only when asked for
    const bool instr = g_decode_trace != nullptr || g_tuning.s_ahead != 4 || g_tuning.l2_ahead != 0;
    const bool mask = npi != nullptr || n_stride % kNT != 0 || h_index != nullptr;
    const bool r16 = rows <= 16 && !instr;  // one beam x <= 16 heads (vchunks == 1)
    auto kern = instr ? (mask ? el_decode_tc_kernel<UNITS, true, true> : el_decode_tc_kernel<UNITS, true, false>)
                : r16 ? (mask ? el_decode_tc_kernel<UNITS, false, true, true> : el_decode_tc_kernel<UNITS, false, false, true>)
                      : (mask ? el_decode_tc_kernel<UNITS, false, true> : el_decode_tc_kernel<UNITS, false, false>);
    constexpr uint32_t smem = DecLayout<UNITS>::kTotal;
    ELA_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    // persistent: one cluster per pair of SMs
    const int max_cl = num_sms_decode() / 2;
    int clusters;
    SplitArgs sa{};
    sa.h_index = h_index;
    // Whole inputs strided over the clusters unless the last round would fill less than 60%
    // of the clusters: then stream-K (every input-segment transition costs a pipeline drain,
    // so splitting only pays when the tail is short; measured on B200 for B = 64..320).
    const int last_round = B % max_cl;
    // ELATTN_DECODE_SCHED = auto (default) | streamk | tail | whole: tuning override
    static const int sched_mode_env = [] {
        const char* e = getenv("ELATTN_DECODE_SCHED");
        if (!e) return 0;
        const std::string v(e);
        return v == "streamk" ? 1 : v == "whole" ? 2 : v == "tail" ? 3 : 0;
    }();
    const int sched_mode = g_decode_sched_override ? g_decode_sched_override : sched_mode_env;
    // H's L2 policy: streamed once (evict-first) unless it fits in L2 with room to spare —
    // then every layer of a decoder step re-reads it from L2 (evict-last; measured 2% per
    // step at B = 16 and 1% at B = 32 (64 MB), worse from 80 MB: tools/time_small_batch.py,
    // profiles/r02c_h_keep_sweep.txt); sibling virtual inputs (> 64 rows) share H_b across
    // neighbouring clusters (evict-normal).
    // ELATTN_DECODE_H_POLICY = auto | first | normal | last, ELATTN_DECODE_H_KEEP_MB (64)
    static const int h_pol_mode = [] {
        const char* e = getenv("ELATTN_DECODE_H_POLICY");
        const std::string v = e ? e : "";
        return v == "first" ? 1 : v == "normal" ? 2 : v == "last" ? 3 : 0;
    }();
    static const size_t h_keep_bytes = [] {
        const char* e = getenv("ELATTN_DECODE_H_KEEP_MB");
        return size_t(e ? atoi(e) : 64) << 20;
    }();
    const size_t h_bytes = size_t(B_h) * n_stride * d_m * 2;
    sa.h_pol = h_pol_mode == 1   ? ptx::kEvictFirst
               : h_pol_mode == 2 ? ptx::kEvictNormal
               : h_pol_mode == 3 ? ptx::kEvictLast
               : h_bytes <= h_keep_bytes ? ptx::kEvictLast
               : vchunks > 1     ? ptx::kEvictNormal
                                 : ptx::kEvictFirst;
    // ragged lengths, moderate batch: stream-K over the inputs' own tile counts (whole-input
    // striding leaves the clusters with the short inputs idle); ELATTN_DECODE_SCHED=whole off
    // ragged lengths: whole inputs, longest first (default); stream-K over the inputs' own tiles
    // only on request (ELATTN_DECODE_SCHED=streamk: splitting costs more than it balances,
    // profiles/r02b_ragged.md)
    const int T_stride = (n_stride + kNT - 1) / kNT;
    const bool ragged_sk = npi != nullptr && sched_mode == 1 && B <= kRaggedSkMaxInputs * max_cl;
    const bool ragged_lpt = npi != nullptr && !ragged_sk && sched_mode != 2 && B > max_cl && T_stride <= kLptMaxTiles &&
                            B < 65536 && (B + max_cl - 1) / max_cl <= kLptMaxList;
    sa.h_pre = (h_static && npi == nullptr && pdl_enabled()) ? std::min(DecLayout<UNITS>::kRing / UNITS, 8) : 0;
    const bool stream_k = npi == nullptr && last_round != 0 &&
                          (sched_mode == 1 || sched_mode == 3 || (sched_mode == 0 && 5 * last_round < 3 * max_cl));
    // TAIL-SPLIT instead of stream-K when there is at least one full round and the leftover
    // inputs, cut into P <= kMaxSegs equal parts, keep >= 3/4 of the clusters busy: the
    // full rounds stay whole inputs (no records, no extra transitions)
    const int T_all = (n_stride + kNT - 1) / kNT;
    const int P_tail = last_round > 0 ? std::min(kMaxSegs, std::min(max_cl / last_round, T_all)) : 0;
    // (also with no full round, B < #clusters: every input in P parts, one segment per
    // cluster — no pipeline transitions, unlike stream-K chunks that straddle inputs)
    // (parts of >= 10 tiles there: shorter parts cost more in records and merging than the
    // transitions they avoid; tools/time_small_batch.py: B = 24 / 32 -6% / -4%, B = 8 +5%)
    const bool tail_split = stream_k && sched_mode != 1 && P_tail >= 2 && (B >= max_cl || T_all >= 10 * P_tail) &&
                            (sched_mode == 3 || 4 * last_round * P_tail >= 3 * max_cl);
    if (ragged_lpt) {
        sa.T = -2;
        sa.vchunks = vchunks;
        clusters = B < max_cl ? B : max_cl;
    } else if (ragged_sk) {
        const int T_all_r = (n_stride + kNT - 1) / kNT;
        sa.T = -1;
        sa.W = std::max(kMinChunkTiles, (T_all_r + kMaxSegs - 2) / (kMaxSegs - 1));  // minimum chunk
        sa.vchunks = vchunks;
        sa.part = part;
        clusters = max_cl;
    } else if (tail_split) {
        sa.T = T_all;
        sa.W = -P_tail;
        sa.vchunks = vchunks;
        clusters = max_cl;
        constexpr size_t kPF = kPartFloatsHdr + size_t(UNITS) * kPartFloatsUnit;
        (void)kPF;
        sa.part = part;
    } else if (stream_k) {
        // stream-K over B*T tiles: chunks of W tiles (>= kMinChunkTiles), one per cluster
        const int T = (n_stride + kNT - 1) / kNT;
        const int64_t TT = int64_t(B) * T;
        int64_t ncl = std::min<int64_t>(max_cl, std::max<int64_t>(1, TT / kMinChunkTiles));
        // chunks of >= T/(kMaxSegs-1) tiles keep every input within kMaxSegs segments
        const int64_t W = std::max<int64_t>((TT + ncl - 1) / ncl, (T + kMaxSegs - 2) / (kMaxSegs - 1));
        ncl = (TT + W - 1) / W;
        ELA_REQUIRE(TT < (int64_t(1) << 30), ELATTN_ERR_UNSUPPORTED, "tcgen05 decode: too many tiles");
        if (W % T != 0) {  // some inputs are split across clusters: partial records
            constexpr size_t kPF = kPartFloatsHdr + size_t(UNITS) * kPartFloatsUnit;
            (void)kPF;
            sa.part = part;
        }
        sa.T = T;
        sa.W = int(W);
        sa.vchunks = vchunks;
        clusters = int(ncl);
    } else {
        sa.T = 0;  // whole inputs, strided over the clusters
        sa.vchunks = vchunks;
        clusters = B < max_cl ? B : max_cl;
    }
    // the kernel is declared with __cluster_dims__(2, 1, 1)
    launch_ex(kern, dim3(2 * clusters), dim3(kThreads), smem, st, 1, tq, th, tc,
              static_cast<const __nv_bfloat16*>(qp), npi, B, rows, n_stride, d_m, scale_log2,
              static_cast<__nv_bfloat16*>(ctx), g_decode_trace, g_tuning, sa, stats, pdl_enabled() ? 1 : 0);
    ELA_CHECK_LAUNCH();
    if (((sa.T > 0 && (sa.W < 0 || sa.W % sa.T != 0)) || sa.T == -1) && clusters > 1) {
        ELA_REQUIRE(part != nullptr, ELATTN_ERR_PARAM, "tcgen05 decode: split schedule needs the partial-record scratch");
        const int Bw = B - last_round;
        const int gx = sa.W < 0 ? last_round : clusters - 1;
        launch_ex(el_decode_merge_kernel<UNITS>, dim3(gx, 2, UNITS), dim3(256), 0, st, 1, static_cast<const float*>(sa.part),
                  sa.T, sa.W, clusters, rows, vchunks, d_m, scale_log2, static_cast<__nv_bfloat16*>(ctx), stats, Bw,
                  npi, B, n_stride);
        ELA_CHECK_LAUNCH();
    }
}

}  // namespace

bool el_decode_tc_supported(int rows_per_input, int d_m) {
    // > 64 rows: as ceil(rows / 64) virtual inputs of up to 64 rows sharing H
    const bool rows_ok = rows_per_input >= 1 && rows_per_input <= 8 * kRowsQ;
    return rows_ok && d_m % 256 == 0 && d_m >= 256 && d_m <= 1024;
}

void launch_el_decode_tc(const void* qp, const void* H, const int* n_per_input, int B, int rows_per_input,
                         int n_stride, int d_m, float scale, void* ctx, cudaStream_t st, float2* stats,
                         float* part, bool h_static, const int* h_index, int h_slots) {
    ELA_REQUIRE(el_decode_tc_supported(rows_per_input, d_m), ELATTN_ERR_UNSUPPORTED,
                "tcgen05 decode: rows <= 512, d_m in {256, 512, 768, 1024}");
    ELA_REQUIRE((reinterpret_cast<uintptr_t>(qp) & 15) == 0 && (reinterpret_cast<uintptr_t>(H) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(ctx) & 15) == 0,
                ELATTN_ERR_PARAM, "tcgen05 decode: q', H and C must be 16-byte aligned");
    const float scale_log2 = scale * 1.4426950408889634f;
    static const bool env_read = [] {
        if (const char* e = getenv("ELATTN_DECODE_S_AHEAD")) g_tuning.s_ahead = atoi(e);
        if (const char* e = getenv("ELATTN_DECODE_L2_AHEAD")) g_tuning.l2_ahead = atoi(e);
        if (const char* e = getenv("ELATTN_DECODE_SKIP_C_STORE")) g_tuning.skip_c_store = atoi(e);
        return true;
    }();
    (void)env_read;
    switch (d_m / 256) {
        case 1: return launch_units<1>(qp, H, n_per_input, B, rows_per_input, n_stride, d_m, scale_log2, ctx, st, stats, part, h_static, h_index, h_slots);
        case 2: return launch_units<2>(qp, H, n_per_input, B, rows_per_input, n_stride, d_m, scale_log2, ctx, st, stats, part, h_static, h_index, h_slots);
        case 3: return launch_units<3>(qp, H, n_per_input, B, rows_per_input, n_stride, d_m, scale_log2, ctx, st, stats, part, h_static, h_index, h_slots);
        default: return launch_units<4>(qp, H, n_per_input, B, rows_per_input, n_stride, d_m, scale_log2, ctx, st, stats, part, h_static, h_index, h_slots);
    }
}

}  // namespace elattn_gpu
