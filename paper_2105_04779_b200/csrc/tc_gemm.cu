// tc_gemm.cu — tcgen05 GEMM family for the projection stages of the bf16 path.
//
//   C[z][m][n] = alpha * sum_k A[z][m][k] * B[z][n][k] + bias[z][n]     (bf16 in/out)
//
// Replaces the reference's CPU matmuls of query expansion (attention.hpp:205-206:
// q.Wq_i + bq_i, then Q_i.Wk_i^T) and of the output projection (:283-288 with
// el_bias_terms :221-231: ctx.Wv_i + bv_i, then .Wo + bo).  Every projection of a layer
// step runs here (no vendor BLAS on the path).
//
// Persistent, warp-specialised.  A CTA owns MT m-subtiles of 128 rows x BN columns that
// share each staged B slice (MT = 2 halves the weight traffic of the per-head V
// projection, whose N = d_k = 64).  Measured on B200 (tools/probes/l2_ingress_probe.cu,
// gemm_ingress_probe.cu): a CTA's TMA ingress is bounded by the number of boxes in flight,
// not by L2 bandwidth — one 16 KB box per ~800 cycles — so every stage moves KBP k-blocks
// per operand in ONE 4-D box (64 x rows x KBP k-blocks, the k-block dimension strided by
// 128 B inside the row-major operand), and the epilogue stores 128-row boxes written by
// four warps together instead of 32-row boxes per warp.
//   warp 0      TMA producer (KBP k-blocks of MT A subtiles + the B slice per stage);
//   warp 1      MMA issuer: tcgen05.mma M=128 N=BN K=16, fp32 accumulators in TMEM,
//               double-buffered so the epilogue of tile t overlaps the MMAs of t+1;
//   warps 2..9  epilogue: two groups of four warps (one per TMEM lane quadrant), group g
//               owns column half g; per 64-column block: tcgen05.ld -> alpha/bias -> bf16
//               -> SWIZZLE_128B stage (128 rows) -> one TMA tensor store (3-D maps, so
//               head-strided outputs such as q' rows r*h + i and V_i columns i*d_k are
//               written in place).
#include "common.cuh"

#include <cstdlib>
#include <string>
#include "kernels.h"
#include "ptx_sm100.cuh"
#include "timeline.cuh"
#include "tmap.h"

namespace elattn_gpu {

int g_gemm_force_bn = 0, g_gemm_force_mt = 0, g_gemm_force_kbp = 0;  // testing / tuning override (0 = auto)
int g_gemm_force_splitk = -1;  // testing / tuning override of the small-M split-K (-1 = auto, 0 = off)
int g_qexp_fused = -1;         // testing / tuning: fused small-batch query expansion (-1 = auto, 0 = off)
unsigned long long* g_gemm_trace = nullptr;                            // testing: timeline of CTA 0
int g_gemm_epilogue_tma = -1;                                          // testing / tuning: 1 TMA stores, 0 st.global, -1 auto

namespace {

constexpr int kBM = 128, kBK = 64;
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;

template <int BN, int MT, int KBP>
struct GemmSmem {
    static constexpr uint32_t kABytes = kBM * kBK * 2;  // one m-subtile, one k-block
    static constexpr uint32_t kBBytes = BN * kBK * 2;   // the B slice, one k-block
    static constexpr uint32_t kStageBytes = KBP * (MT * kABytes + kBBytes);
    // epilogue: per group (column half) blocks of 128 rows x kPiece columns
    // (64 -> SWIZZLE_128B, 32 -> SWIZZLE_64B)
    static constexpr int kHalf = BN / 2;
    static constexpr int kPiece = kHalf < 64 ? kHalf : 64;
    static constexpr uint32_t kPieceBytes = kBM * kPiece * 2;
    static constexpr uint32_t kFixedNoOut = 256 + 1024;
    // store buffers per group: a TMA store holds its buffer for ~600 ns (until it has read
    // it), so the write-bound shape (BN = 256, one k-step per tile: q' expansion) keeps four
    // in flight per group and two operand stages; the others two, or one if that would
    // leave fewer than three operand stages
    static constexpr int kStages2 = int((232448u - kFixedNoOut - 2 * 2 * kPieceBytes) / kStageBytes);
    static constexpr int kOutBufs = (BN == 256 && KBP == 1) ? 4 : (kStages2 >= 3 ? 2 : 1);
    static constexpr uint32_t kOutBytes = 2 * kOutBufs * kPieceBytes;
    static constexpr int kStagesFit = int((232448u - kFixedNoOut - kOutBytes) / kStageBytes);
    static constexpr int kStages = kStagesFit < 8 ? kStagesFit : 8;
    static constexpr uint32_t kOutOff = kStages * kStageBytes;
    static constexpr uint32_t kBarOff = kOutOff + kOutBytes;
    static constexpr uint32_t kTotal = kBarOff + 256 + 1024;  // + barriers + alignment slack
    static constexpr uint32_t kAccCols = MT * BN;              // one accumulator set
    static constexpr uint32_t kTmemCols =
        2 * kAccCols <= 64 ? 64 : (2 * kAccCols <= 128 ? 128 : (2 * kAccCols <= 256 ? 256 : 512));
    static_assert(2 * kAccCols <= 512, "TMEM: two accumulator sets");
    static_assert(kStages >= 2, "smem ring");
    static_assert(kTotal <= 232448, "smem");
};

struct GemmParams {
    int M, N, K, Z;
    int tiles_m, tiles_n;  // tiles_m counts MT-subtile groups of 128 rows
    float alpha;
    const float* bias;
    int64_t sbz;
    int a_zm, b_zm, c_zm;  // 1: tensor map coordinate order is (k, z, m, ..) instead of (k, m, z, ..)
    int a_bcast;           // A shared by every z (sAz == 0): load it with z = 0
    int pdl;               // wait for the preceding kernel (programmatic dependent launch)
    int direct;            // epilogue: coalesced st.global through a per-warp smem transpose (1) or TMA stores (0)
    __nv_bfloat16* C;      // output for the direct epilogue: C + z * sCz + m * ldc + n
    int64_t ldc, sCz;
    unsigned long long* trace;  // testing: %globaltimer stamps of CTA 0 (null = off)
    uint64_t b_pol;             // L2 policy of the B (weight) loads
    int b_pre;                  // stages of the first tile whose B slice is loaded before the PDL wait
    uint64_t c_pol;             // L2 policy of the TMA-store epilogue's output
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ uint32_t pack2(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ void group_bar(uint32_t id) { asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory"); }

template <int BN, int MT, int KBP, bool BIAS, bool SCALE>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, GemmParams p) {
    ELA_TL_DECL;
    using S = GemmSmem<BN, MT, KBP>;
    constexpr int kStages = S::kStages;
    extern __shared__ uint8_t smem_raw[];
    // 1024-B alignment for SWIZZLE_128B, by offsetting the __shared__ array itself so
    // the compiler keeps the shared address space (LDS/STS, not generic LD/ST)
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* out_stage = smem + S::kOutOff;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kBarOff);
    uint64_t* empty = full + kStages;
    uint64_t* acc_full = empty + kStages;  // [2] MMA -> epilogue
    uint64_t* acc_empty = acc_full + 2;    // [2] epilogue -> MMA
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

    const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
    const bool tr = p.trace != nullptr && blockIdx.x == 0;
    if (tr && threadIdx.x == 0) p.trace[0] = gtimer();
    const int num_kb = p.K / kBK;
    const int num_ks = (num_kb + KBP - 1) / KBP;  // stages per tile (the last may run past K: zero-filled)
    const int num_tiles = p.Z * p.tiles_m * p.tiles_n;
    // z (head) fastest: the CTAs running concurrently touch the SAME rows r of the
    // head-interleaved layouts (q' / C rows r*h + i), so their row pieces land in the same
    // DRAM pages; then n, so neighbouring CTAs share the A rows in L2.  Row blocks run LAST
    // to FIRST: the first inputs' rows are written last and are still in L2 when the next
    // kernel (the decode, reading q' input by input) starts with them
    auto tile_coords = [&](int t, int& z, int& m0, int& n0) {
        z = t % p.Z;
        const int r = t / p.Z;
        m0 = (p.tiles_m - 1 - r / p.tiles_n) * (MT * kBM);
        n0 = (r % p.tiles_n) * BN;
    };

    if (warp == 0) {
        if (ptx::elect_one()) {
            ptx::prefetch_tmap(&tmA);
            ptx::prefetch_tmap(&tmB);
            ptx::prefetch_tmap(&tmC);
            for (int s = 0; s < kStages; ++s) {
                ptx::mbar_init(&full[s], 1);
                ptx::mbar_init(&empty[s], 1);
            }
            for (int i = 0; i < 2; ++i) {
                ptx::mbar_init(&acc_full[i], 1);
                ptx::mbar_init(&acc_empty[i], kEpiWarps);
            }
            ptx::fence_mbar_init();
        }
        __syncwarp();
    } else if (warp == 1) {
        ptx::tmem_alloc<S::kTmemCols>(tmem_slot);
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // weights (B) are never written by the preceding kernels: the producer issues the first
    // stages' B slices BEFORE the programmatic-dependent-launch wait, so their latency
    // overlaps the previous kernel's tail (A, written by it, follows after the wait)
    const int b_pre = (p.pdl && int(blockIdx.x) < num_tiles) ? p.b_pre : 0;
    if (p.pdl) {
        // prologue done (TMEM held): the next kernel may launch; wait for the previous one
        ptx::griddep_launch_dependents();
        if (warp == 0 && b_pre > 0 && ptx::elect_one()) {
            int z, m0, n0;
            tile_coords(int(blockIdx.x), z, m0, n0);
            for (int s = 0; s < b_pre; ++s) {
                uint8_t* b = smem + s * S::kStageBytes + KBP * MT * S::kABytes;
                ptx::mbar_arrive_expect_tx(&full[s], S::kStageBytes);
                if (p.b_zm)
                    ptx::tma_load_4d(b, &tmB, &full[s], 0, z, n0, s * KBP, p.b_pol);
                else
                    ptx::tma_load_4d(b, &tmB, &full[s], 0, n0, z, s * KBP, p.b_pol);
            }
        }
        __syncwarp();
        ptx::griddep_wait();
        ELA_TL_WAIT();
    }
    if (tr && threadIdx.x == 0) p.trace[1] = gtimer();

    if (warp == 0) {
        // ---- TMA producer: per stage one 4-D box per A subtile and one for B
        if (ptx::elect_one()) {
            int it = 0;
            for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
                int z, m0, n0;
                tile_coords(t, z, m0, n0);
                const int za = p.a_bcast ? 0 : z;
                for (int ks = 0; ks < num_ks; ++ks, ++it) {
                    const int s = it % kStages;
                    ptx::mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
                    uint8_t* a = smem + s * S::kStageBytes;
                    uint8_t* b = a + KBP * MT * S::kABytes;
                    const bool pre = it < b_pre;  // B already in flight (issued before the PDL wait)
                    if (!pre) ptx::mbar_arrive_expect_tx(&full[s], S::kStageBytes);
                    const int kb = ks * KBP;
                    if (tr && it < 4) p.trace[52 + it] = gtimer();
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) {
                        uint8_t* dst = a + mt * KBP * S::kABytes;  // [kb][128 rows][64]
                        if (p.a_zm)
                            ptx::tma_load_4d(dst, &tmA, &full[s], 0, za, m0 + mt * kBM, kb, ptx::kEvictNormal);
                        else
                            ptx::tma_load_4d(dst, &tmA, &full[s], 0, m0 + mt * kBM, za, kb, ptx::kEvictNormal);
                    }
                    if (!pre) {
                        if (p.b_zm)
                            ptx::tma_load_4d(b, &tmB, &full[s], 0, z, n0, kb, p.b_pol);
                        else
                            ptx::tma_load_4d(b, &tmB, &full[s], 0, n0, z, kb, p.b_pol);
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ---- MMA issuer (whole warp loops; lane 0 issues and commits)
        constexpr uint32_t idesc = ptx::idesc_bf16(kBM, BN, 0, 0);
        const uint64_t d0 = ptx::sdesc_sw128(ptx::smem_u32(smem), 0, 1024);
        int it = 0, local = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++local) {
            const int ab = local & 1;
            ptx::mbar_wait(&acc_empty[ab], ((local >> 1) & 1) ^ 1);
            ptx::tc_fence_after();
            const uint32_t d = tmem + ab * S::kAccCols;
            for (int ks = 0; ks < num_ks; ++ks, ++it) {
                const int s = it % kStages;
                ptx::mbar_wait(&full[s], (it / kStages) & 1);
                if (it == 0 && lane == 0) ELA_TL_MARK(0);  // first stage landed
                ptx::tc_fence_after();
                if (tr && lane == 0 && it < 32) p.trace[2 + it] = gtimer();
                if (lane == 0) {
                    const uint64_t a = d0 + uint64_t((s * S::kStageBytes) >> 4);
                    const uint64_t b = a + uint64_t((KBP * MT * S::kABytes) >> 4);
                    const int nk = min(KBP, num_kb - ks * KBP);
#pragma unroll
                    for (int j = 0; j < KBP; ++j) {
                        if (j >= nk) break;
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                            for (int k = 0; k < kBK / 16; ++k)
                                ptx::mma_bf16(d + mt * BN,
                                              a + uint64_t(((mt * KBP + j) * S::kABytes) >> 4) + uint64_t(2 * k),
                                              b + uint64_t((j * S::kBBytes) >> 4) + uint64_t(2 * k), idesc,
                                              (ks | j | k) != 0);
                    }
                    ptx::mma_commit(&empty[s]);
                }
                __syncwarp();
            }
            if (lane == 0) ptx::mma_commit(&acc_full[ab]);
            __syncwarp();
        }
    } else {
        // ---- epilogue: group g = column half (warps 2..5 -> 0, 6..9 -> 1); within a group
        // warp w reads TMEM lane quadrant qd = w % 4 (rows 32 qd ..).  Per block of kPiece
        // columns the four warps fill one 128-row stage and warp (w - 2) % 4 == 0 stores it.
        const uint32_t qd = warp & 3, grp = (warp - 2) >> 2;
        const bool leader = ((warp - 2) & 3) == 0 && lane == 0;
        constexpr int kHalf = S::kHalf, kPiece = S::kPiece;
        uint8_t* grp_stage = out_stage + grp * S::kOutBufs * S::kPieceBytes;
        const uint32_t bar_id = 1 + grp;
        int local = 0, piece = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++local) {
            int z, m0, n0;
            tile_coords(t, z, m0, n0);
            const int ab = local & 1;
            // bias of this warp's columns (lane l: column 32 c + l of the half), loaded
            // before the accumulator is ready
            float bcol[kHalf / 32];
            if constexpr (BIAS) {
#pragma unroll
                for (int c = 0; c < kHalf / 32; ++c) {
                    const int n = n0 + int(grp) * kHalf + 32 * c + int(lane);
                    bcol[c] = n < p.N ? __ldg(p.bias + z * p.sbz + n) : 0.f;
                }
            }
            ptx::mbar_wait(&acc_full[ab], (local >> 1) & 1);
            if (warp == 2 && lane == 0) ELA_TL_MARK(1);  // (last) accumulator ready
            ptx::tc_fence_after();
            if (tr && warp == 2 && lane == 0 && local < 8) p.trace[34 + 2 * local] = gtimer();
#pragma unroll 1
            for (int mt = 0; mt < MT; ++mt) {
#pragma unroll 1
                for (int c0 = 0; c0 < kHalf; c0 += kPiece, ++piece) {
                    const uint32_t t_row =
                        tmem + ((qd * 32) << 16) + ab * S::kAccCols + mt * BN + grp * kHalf + c0;
                    uint32_t rr[kPiece];
#pragma unroll
                    for (int c = 0; c < kPiece; c += 32)
                        ptx::tmem_ld32(t_row + c, *reinterpret_cast<uint32_t(*)[32]>(&rr[c]));
                    ptx::tmem_ld_wait();
                    if (tr && warp == 2 && lane == 0 && piece < 2) p.trace[60 + 3 * piece] = gtimer();
                    if (mt == MT - 1 && c0 + kPiece >= kHalf) {
                        // this warp's part of the accumulator is read: the MMA warp may reuse it
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) ptx::mbar_arrive(&acc_empty[ab]);
                    }
                    uint8_t* stage = grp_stage + (piece % S::kOutBufs) * S::kPieceBytes;
                    if (!p.direct) {
                        // the store that last used this buffer has read it
                        if (leader) ptx::bulk_wait_group_read<S::kOutBufs - 1>();
                        group_bar(bar_id);
                    }
#pragma unroll
                    for (int cc = 0; cc < kPiece; cc += 32) {
                        uint32_t packed[16];
#pragma unroll
                        for (int j = 0; j < 32; j += 2) {
                            float v0 = __uint_as_float(rr[cc + j]), v1 = __uint_as_float(rr[cc + j + 1]);
                            if constexpr (SCALE) v0 *= p.alpha, v1 *= p.alpha;
                            if constexpr (BIAS) {
                                const float bc = bcol[(c0 + cc) / 32];
                                v0 += __shfl_sync(0xffffffffu, bc, j);
                                v1 += __shfl_sync(0xffffffffu, bc, j + 1);
                            }
                            packed[j / 2] = pack2(v0, v1);
                        }
                        // row 32 qd + lane: SWIZZLE_128B (16-byte chunk c of row l at c ^ (l & 7))
                        // for 64-column blocks, SWIZZLE_64B (c ^ ((l >> 1) & 3)) for 32
                        uint8_t* row = stage + (qd * 32 + lane) * (kPiece * 2);
                        const int cbase = cc >> 3;
                        const int sw = kPiece == 64 ? int(lane & 7) : int((lane >> 1) & 3);
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            *reinterpret_cast<uint4*>(row + (((cbase + q) ^ sw) << 4)) =
                                make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
                    }
                    if (p.direct) {
                        // this warp's 32 rows leave through its own slice of the stage,
                        // read back row-contiguous: each st.global.v4 instruction writes
                        // 32 / kChunks whole 128-byte (64-byte) row pieces
                        constexpr int kChunks = kPiece / 8, kRowsPerInst = 32 / kChunks;
                        __syncwarp();
                        if (tr && warp == 2 && lane == 0 && piece < 2) p.trace[61 + 3 * piece] = gtimer();
                        const uint8_t* slice = stage + qd * 32 * (kPiece * 2);
                        const int rbase = m0 + mt * kBM + int(qd) * 32, cbase = n0 + int(grp) * kHalf + c0;
#pragma unroll
                        for (int s = 0; s < 32 / kRowsPerInst; ++s) {
                            const int rr = s * kRowsPerInst + int(lane) / kChunks, ch = int(lane) % kChunks;
                            const int sw = kPiece == 64 ? (rr & 7) : ((rr >> 1) & 3);
                            const uint4 v = *reinterpret_cast<const uint4*>(slice + rr * (kPiece * 2) + ((ch ^ sw) << 4));
                            const int row = rbase + rr, col = cbase + ch * 8;
                            if (row < p.M && col < p.N)
                                *reinterpret_cast<uint4*>(p.C + z * p.sCz + int64_t(row) * p.ldc + col) = v;
                        }
                        __syncwarp();
                        if (tr && warp == 2 && lane == 0 && piece < 2) p.trace[62 + 3 * piece] = gtimer();
                        continue;
                    }
                    ptx::fence_proxy_async_smem();
                    group_bar(bar_id);
                    if (tr && leader && warp == 2 && piece < 4) p.trace[56 + piece] = gtimer();
                    if (leader) {
                        const int nbase = n0 + int(grp) * kHalf + c0, r0 = m0 + mt * kBM;
                        if (nbase < p.N && r0 < p.M) {
                            if (p.c_zm)
                                ptx::tma_store_3d_hint(&tmC, stage, nbase, z, r0, p.c_pol);
                            else
                                ptx::tma_store_3d_hint(&tmC, stage, nbase, r0, z, p.c_pol);
                        }
                        ptx::bulk_commit_group();
                    }
                }
            }
        }
        // the smem stages must stay valid until the stores have read them (global
        // visibility of TMA stores is guaranteed at grid completion)
        if (leader) ptx::bulk_wait_group_read<0>();
        __syncwarp();
        if (tr && warp == 2 && lane == 0) p.trace[50] = gtimer();
        if (warp == 2 && lane == 0) ELA_TL_MARK(2);  // epilogue done
    }
    ptx::tc_fence_before();
    __syncthreads();
    ELA_TL_EXIT(kTlGemm);
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<S::kTmemCols>(tmem);
    }
}

// ---------------------------------------------------------------- split-K (small M)
// For the projections of a SMALL batch (M = B*x rows <= a few hundred) the tile grid
// above has 8-16 CTAs, each streaming the whole K through one TMA engine: latency-bound
// (~9 us for a 128 x 1024 x 1024 GEMM).  Here a CLUSTER of SK CTAs shares one 128 x 64
// output tile: CTA r multiplies k-blocks [r*nkb/SK, (r+1)*nkb/SK) (one TMA box per
// operand, all in flight at once), then the partial accumulators are REDUCE-SCATTERED
// through DSMEM: CTA r owns columns [r*W, (r+1)*W) (W = 64/SK), receives those columns
// of the other SK-1 partials (st.async + mbarrier complete_tx) and sums all SK in rank
// order (deterministic), adds the bias and stores bf16.
//   warp 0: TMA (A and B boxes of this CTA's k-slice); warp 1: TMEM owner + MMA issuer;
//   warps 2..5: TMEM lane quadrants (rows 32 qd ..): exchange, reduction, epilogue.
constexpr int kSkBN = 64;
constexpr int kSkThreads = 192;

struct SkParams {
    int M, N, K, Z, tiles_m, tiles_n, kbp, a_zm, b_zm, a_bcast, pdl, b_static;
    float alpha;
    const float* bias;
    int64_t sbz;
    __nv_bfloat16* C;
    int64_t ldc, sCz;
};

template <int SK>
struct SkSmem {
    static constexpr int kW = kSkBN / SK;  // columns owned per CTA
    static constexpr uint32_t kRecvBytes = uint32_t(SK - 1) * kBM * kW * 4;
    static constexpr uint32_t kMaxKbp = 8;
    static constexpr uint32_t kABytes = kBM * kBK * 2, kBBytes = kSkBN * kBK * 2;
    static constexpr uint32_t kBOff = kMaxKbp * kABytes;
    static constexpr uint32_t kRecvOff = kBOff + kMaxKbp * kBBytes;
    static constexpr uint32_t kBarOff = kRecvOff + kRecvBytes;
    static constexpr uint32_t kTotal = kBarOff + 64 + 1024;
    static_assert(kTotal <= 232448, "split-K shared memory");
};

template <int SK, bool BIAS, bool SCALE>
__global__ void __launch_bounds__(kSkThreads, 1)
    tc_gemm_splitk_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                          SkParams p) {
    ELA_TL_DECL;
    using S = SkSmem<SK>;
    constexpr int kW = S::kW;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;
    uint8_t* sB = smem + S::kBOff;
    float* recv = reinterpret_cast<float*>(smem + S::kRecvOff);  // [SK-1][128 rows][kW]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kBarOff);
    uint64_t* acc_full = full + 1;
    uint64_t* recv_full = full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(full + 3);
    const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
    const int rank = int(ptx::cluster_ctarank());
    const int t = int(blockIdx.x) / SK;
    const int z = t % p.Z, r_ = t / p.Z;
    const int m0 = (r_ / p.tiles_n) * kBM, n0 = (r_ % p.tiles_n) * kSkBN;
    const int kb0 = rank * p.kbp;

    if (warp == 0) {
        if (ptx::elect_one()) {
            ptx::prefetch_tmap(&tmA);
            ptx::prefetch_tmap(&tmB);
            ptx::mbar_init(full, 1);
            ptx::mbar_init(acc_full, 1);
            ptx::mbar_init(recv_full, 1);
            ptx::fence_mbar_init();
            // the peers' partial columns may arrive before this CTA reaches its wait
            if (SK > 1) ptx::mbar_arrive_expect_tx(recv_full, S::kRecvBytes);
        }
        __syncwarp();
    } else if (warp == 1) {
        ptx::tmem_alloc<64>(tmem_slot);
    }
    ptx::tc_fence_before();
    ptx::cluster_sync();  // barriers initialised before any peer st.async targets them
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const bool b_early = p.pdl && p.b_static;  // weights: fetched before the PDL wait
    if (p.pdl) {
        ptx::griddep_launch_dependents();
        if (warp == 0 && b_early && ptx::elect_one()) {
            ptx::mbar_arrive_expect_tx(full, uint32_t(p.kbp) * (S::kABytes + S::kBBytes));
            if (p.b_zm)
                ptx::tma_load_4d(sB, &tmB, full, 0, z, n0, kb0, ptx::kEvictLast);
            else
                ptx::tma_load_4d(sB, &tmB, full, 0, n0, z, kb0, ptx::kEvictLast);
        }
        __syncwarp();
        ptx::griddep_wait();
        ELA_TL_WAIT();
    }
    if (warp == 0) {
        if (ptx::elect_one()) {
            if (!b_early) ptx::mbar_arrive_expect_tx(full, uint32_t(p.kbp) * (S::kABytes + S::kBBytes));
            const int za = p.a_bcast ? 0 : z;
            if (p.a_zm)
                ptx::tma_load_4d(sA, &tmA, full, 0, za, m0, kb0, ptx::kEvictNormal);
            else
                ptx::tma_load_4d(sA, &tmA, full, 0, m0, za, kb0, ptx::kEvictNormal);
            if (!b_early) {
                if (p.b_zm)
                    ptx::tma_load_4d(sB, &tmB, full, 0, z, n0, kb0, ptx::kEvictLast);
                else
                    ptx::tma_load_4d(sB, &tmB, full, 0, n0, z, kb0, ptx::kEvictLast);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        constexpr uint32_t idesc = ptx::idesc_bf16(kBM, kSkBN, 0, 0);
        ptx::mbar_wait(full, 0);
        if (lane == 0) ELA_TL_MARK(0);  // operands landed
        ptx::tc_fence_after();
        if (lane == 0) {
            const uint64_t a0 = ptx::sdesc_sw128(ptx::smem_u32(sA), 0, 1024);
            const uint64_t b0 = ptx::sdesc_sw128(ptx::smem_u32(sB), 0, 1024);
            for (int j = 0; j < p.kbp; ++j)
#pragma unroll
                for (int k = 0; k < kBK / 16; ++k)
                    ptx::mma_bf16(tmem, a0 + uint64_t((j * S::kABytes) >> 4) + uint64_t(2 * k),
                                  b0 + uint64_t((j * S::kBBytes) >> 4) + uint64_t(2 * k), idesc, (j | k) != 0);
            ptx::mma_commit(acc_full);
        }
        __syncwarp();
    } else {
        const uint32_t qd = warp & 3;
        const int row = int(qd) * 32 + int(lane), m = m0 + row;
        float bcol[kW];
#pragma unroll
        for (int j = 0; j < kW; ++j) {
            const int n = n0 + rank * kW + j;
            bcol[j] = (BIAS && n < p.N) ? __ldg(p.bias + z * p.sbz + n) : 0.f;
        }
        ptx::mbar_wait(acc_full, 0);
        if (warp == 2 && lane == 0) ELA_TL_MARK(1);  // accumulator ready
        ptx::tc_fence_after();
        uint32_t v[64];
        ptx::tmem_ld32(tmem + ((qd * 32) << 16), *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
        ptx::tmem_ld32(tmem + ((qd * 32) << 16) + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
        ptx::tmem_ld_wait();
        if constexpr (SK == 2) {
            // one peer: this row's other 32-column half goes straight from registers (st.async;
            // the loop keeps the register indices compile-time)
#pragma unroll
            for (int pr = 0; pr < SK; ++pr) {
                if (pr == rank) continue;
                const uint32_t dst = ptx::mapa(ptx::smem_u32(recv + row * kW), uint32_t(pr));
                const uint32_t bar = ptx::mapa(ptx::smem_u32(recv_full), uint32_t(pr));
#pragma unroll
                for (int j = 0; j < kW; j += 4)
                    ptx::st_async_v4(dst + 4 * j, __uint_as_float(v[pr * kW + j]), __uint_as_float(v[pr * kW + j + 1]),
                                     __uint_as_float(v[pr * kW + j + 2]), __uint_as_float(v[pr * kW + j + 3]), bar);
            }
            ptx::mbar_wait(recv_full, 0);
            if (warp == 2 && lane == 0) ELA_TL_MARK(2);  // peer's partial columns received
        } else if constexpr (SK > 2) {
            // column slice p of the partial goes to CTA p (slot = this CTA's index among p's
            // sources): staged as [p][128 rows][kW] in the A operand region (the MMAs that read
            // it have completed), then ONE bulk shared::cta -> shared::cluster copy per peer
            // (per-row st.async of 16 bytes made this exchange ~0.5 us slower at SK = 4)
            float* send = reinterpret_cast<float*>(sA);
#pragma unroll
            for (int pr = 0; pr < SK; ++pr) {
                if (pr == rank) continue;
#pragma unroll
                for (int j = 0; j < kW; j += 4)
                    *reinterpret_cast<float4*>(send + (pr * kBM + row) * kW + j) =
                        make_float4(__uint_as_float(v[pr * kW + j]), __uint_as_float(v[pr * kW + j + 1]),
                                    __uint_as_float(v[pr * kW + j + 2]), __uint_as_float(v[pr * kW + j + 3]));
            }
            ptx::fence_proxy_async_smem();
            asm volatile("bar.sync 1, 128;" ::: "memory");  // the four epilogue warps staged their rows
            if (warp == 2 && lane == 0) {
#pragma unroll
                for (int pr = 0; pr < SK; ++pr) {
                    if (pr == rank) continue;
                    const int slot = rank - (rank > pr ? 1 : 0);
                    ptx::bulk_s2s_cluster(ptx::mapa(ptx::smem_u32(recv + slot * kBM * kW), uint32_t(pr)),
                                          ptx::smem_u32(send + pr * kBM * kW), uint32_t(kBM * kW * 4),
                                          ptx::mapa(ptx::smem_u32(recv_full), uint32_t(pr)));
                }
            }
            ptx::mbar_wait(recv_full, 0);
            if (warp == 2 && lane == 0) ELA_TL_MARK(2);  // peers' partial columns received
        }
        float acc[kW];
#pragma unroll
        for (int j = 0; j < kW; ++j) acc[j] = 0.f;
#pragma unroll
        for (int sr = 0; sr < SK; ++sr) {  // rank order: deterministic
            if (sr == rank) {
#pragma unroll
                for (int j = 0; j < kW; ++j) acc[j] += __uint_as_float(v[rank * kW + j]);
            } else {
                const float* src = recv + ((sr - (sr > rank ? 1 : 0)) * kBM + row) * kW;
#pragma unroll
                for (int j = 0; j < kW; ++j) acc[j] += src[j];
            }
        }
        if (m < p.M) {
            __nv_bfloat16* dst = p.C + z * p.sCz + int64_t(m) * p.ldc + n0 + rank * kW;
#pragma unroll
            for (int j = 0; j < kW; j += 8) {
                if (n0 + rank * kW + j + 8 > p.N) break;
                uint4 o;
                float f[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) f[i] = (SCALE ? acc[j + i] * p.alpha : acc[j + i]) + bcol[j + i];
                o.x = pack2(f[0], f[1]);
                o.y = pack2(f[2], f[3]);
                o.z = pack2(f[4], f[5]);
                o.w = pack2(f[6], f[7]);
                *reinterpret_cast<uint4*>(dst + j) = o;
            }
        }
        if (warp == 2 && lane == 0) ELA_TL_MARK(3);  // stores issued
    }
    ptx::tc_fence_before();
    // no CTA leaves while its partial columns are still in flight to a peer: each peer waited
    // for all of its incoming columns (recv_full) before arriving, so an execution barrier is
    // enough (a release would first drain this CTA's C stores, ~1 us)
    ptx::cluster_sync_relaxed();
    ELA_TL_EXIT(kTlSplitK);
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<64>(tmem);
    }
}

// ---------------------------------------------------------------- fused query expansion (small M)
// q'_{r,i} = (y_r . W_Q,i + b_Q,i) . W_K,i^T for a small batch in ONE launch (replaces the Q
// GEMM + the head-batched q' GEMM, both latency-bound at a few hundred rows).  CTA
// (128-row tile, head i, quarter u):
//   1. the whole Q_i tile (128 x 64, K = d_m) on the tensor cores, Y and W_Q,i streamed in
//      3 stages of 2 k-blocks (the W_Q,i stages are issued before the PDL wait);
//   2. Q_i + b_Q,i -> bf16 -> this CTA's shared memory as the SW128 K-major A operand;
//   3. the CTA's quarter of d_m: q'[rows][d_m u / 4 ..) = Q_i . W_K,i^T in 128-column chunks
//      (M128 N128 K64), stored straight to the q' rows r*h + i.
// The four quarters recompute Q_i (the Y tile and W_Q,i are L2 hits) instead of splitting K
// over a cluster: the DSMEM reduce-scatter + all-gather that version needed cost ~4 us of
// latency, more than the recomputation (a CTA-pair variant that multicast each stage's two
// k-blocks, halving the L2 requests, measured slower: the single-k-block boxes).  Q is
// rounded to bf16 before step 3 and accumulated over K in one chain, as the two-kernel path
// does, so the result is bit-identical to it.  Standalone (graph replay, beam 4): 7.0 us at
// B <= 16 vs 9.1 for the two GEMMs; 8.3 vs 8.5 at B = 32, where the two-GEMM path is still
// ahead inside the decoder step (the split-K Q GEMM spreads the 256 KB Y tile over 4 CTAs)
// Four k-blocks per TMA box (64 KB Y / 32 KB W_Q boxes: a CTA's TMA ingress grows with the
// box size, tools/probes/gemm_ingress_probe.cu) in two stages; the second W_K chunk buffer
// is stage 0's memory, free once the Q_i accumulation has drained.
constexpr int kQxThreads = 192, kQxKbp = 4, kQxStages = 2;
struct QxSmem {
    static constexpr uint32_t kABytes = kBM * kBK * 2;  // Y: 128 rows x 64 k
    static constexpr uint32_t kBBytes = 64 * kBK * 2;   // W_Q,i: 64 rows x 64 k
    static constexpr uint32_t kStageBytes = kQxKbp * (kABytes + kBBytes);
    static constexpr uint32_t kWkBytes = 128 * 64 * 2;           // one W_K chunk: 128 rows x 64 k
    static constexpr uint32_t kQOff = kQxStages * kStageBytes;  // Q_i bf16, 128 x 64, SW128 K-major
    static constexpr uint32_t kWkOff = kQOff + kBM * 64 * 2;    // W_K chunk buffer 0 (buffer 1: stage 0)
    static constexpr uint32_t kBarOff = kWkOff + kWkBytes;
    static constexpr uint32_t kTotal = kBarOff + 256 + 1024;
    static_assert(kTotal <= 232448, "fused query expansion shared memory");
    static_assert(kStageBytes >= kWkBytes, "W_K chunk buffer 1 lives in stage 0");
};
struct QxParams {
    int M, d_m, h, nkb, nks, chunks, pdl;  // chunks: 128-column q' chunks per CTA (d_m / 4 / 128)
    const float* bq;
    __nv_bfloat16* qp;                     // [M * h][d_m]
};

__global__ void __launch_bounds__(kQxThreads, 1)
    tc_qexp_kernel(const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmWq,
                   const __grid_constant__ CUtensorMap tmWk, QxParams p) {
    ELA_TL_DECL;
    using S = QxSmem;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sQ = smem + S::kQOff;
    uint8_t* sWk = smem + S::kWkOff;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kBarOff);  // [kQxStages]
    uint64_t* empty = full + kQxStages;                                // [kQxStages]
    uint64_t* acc_full = empty + kQxStages;
    uint64_t* q_full = acc_full + 1;   // epilogue warps -> MMA: Q_i staged in sQ
    uint64_t* wk_full = q_full + 1;    // [2]
    uint64_t* p_full = wk_full + 2;    // [2]
    uint64_t* p_empty = p_full + 2;    // [2] (epilogue -> MMA: q' chunk accumulator read)
    uint64_t* wk_empty = p_empty + 2;  // [2] (MMA -> TMA: W_K chunk buffer consumed)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wk_empty + 2);
    const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
    const int quarter = int(blockIdx.x) & 3, t = int(blockIdx.x) >> 2;
    const int z = t % p.h, m0 = (t / p.h) * kBM;  // quarter, then head fastest: neighbours share Y rows in L2
    const int col0 = quarter * (p.d_m / 4);      // this CTA's q' columns
    auto stage_a = [&](int s) { return smem + s * S::kStageBytes; };
    auto stage_b = [&](int s) { return smem + s * S::kStageBytes + kQxKbp * S::kABytes; };

    if (warp == 0) {
        if (ptx::elect_one()) {
            ptx::prefetch_tmap(&tmY);
            ptx::prefetch_tmap(&tmWq);
            ptx::prefetch_tmap(&tmWk);
            for (int s = 0; s < kQxStages; ++s) {
                ptx::mbar_init(&full[s], 1);
                ptx::mbar_init(&empty[s], 1);
            }
            ptx::mbar_init(acc_full, 1);
            ptx::mbar_init(q_full, 4);
            for (int i = 0; i < 2; ++i) {
                ptx::mbar_init(&wk_full[i], 1);
                ptx::mbar_init(&p_full[i], 1);
                ptx::mbar_init(&p_empty[i], 4);
                ptx::mbar_init(&wk_empty[i], 1);
            }
            ptx::fence_mbar_init();
        }
        __syncwarp();
    } else if (warp == 1) {
        ptx::tmem_alloc<512>(tmem_slot);
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tq = tmem, tp = tmem + 128;  // Q_i: 64 columns; q' chunks: 2 x 128 columns
    const int b_pre = p.pdl ? min(kQxStages, p.nks) : 0;
    auto wk_buf = [&](int bi) { return bi == 0 ? sWk : smem; };  // buffer 1 = stage 0 (after phase 1)
    auto load_wk = [&](int c) {
        const int bi = c & 1;
        ptx::mbar_arrive_expect_tx(&wk_full[bi], S::kWkBytes);
        ptx::tma_load_3d(wk_buf(bi), &tmWk, &wk_full[bi], 0, col0 + c * 128, z, ptx::kEvictLast);
    };
    if (p.pdl) {
        ptx::griddep_launch_dependents();
        // the weights do not depend on the preceding kernels: issue them before the wait
        if (warp == 0 && ptx::elect_one()) {
            for (int s = 0; s < b_pre; ++s) {
                ptx::mbar_arrive_expect_tx(&full[s], S::kStageBytes);
                ptx::tma_load_4d(stage_b(s), &tmWq, &full[s], 0, z * 64, 0, s * kQxKbp, ptx::kEvictLast);
            }
            if (p.chunks > 0) load_wk(0);
        }
        __syncwarp();
        ptx::griddep_wait();
        ELA_TL_WAIT();
    }
    if (warp == 0) {
        if (ptx::elect_one()) {
            if (!p.pdl && p.chunks > 0) load_wk(0);
            for (int ks = 0; ks < p.nks; ++ks) {
                const int s = ks % kQxStages;
                ptx::mbar_wait(&empty[s], ((ks / kQxStages) & 1) ^ 1);
                const bool pre = ks < b_pre;  // W_Q slice already in flight
                if (!pre) ptx::mbar_arrive_expect_tx(&full[s], S::kStageBytes);
                ptx::tma_load_4d(stage_a(s), &tmY, &full[s], 0, m0, 0, ks * kQxKbp, ptx::kEvictNormal);
                if (!pre) ptx::tma_load_4d(stage_b(s), &tmWq, &full[s], 0, z * 64, 0, ks * kQxKbp, ptx::kEvictLast);
            }
            // chunk 1 goes to stage 0's memory once every phase-1 MMA has completed
            if (p.chunks > 1) {
                ptx::mbar_wait(acc_full, 0);
                load_wk(1);
            }
            for (int c = 2; c < p.chunks; ++c) {
                ptx::mbar_wait(&wk_empty[c & 1], ((c >> 1) - 1) & 1);
                load_wk(c);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // phase 1: Q_i over the whole K (one accumulation chain, k-blocks in order)
        constexpr uint32_t idq = ptx::idesc_bf16(kBM, 64, 0, 0);
        const uint64_t d0 = ptx::sdesc_sw128(ptx::smem_u32(smem), 0, 1024);
        for (int ks = 0; ks < p.nks; ++ks) {
            const int s = ks % kQxStages;
            ptx::mbar_wait(&full[s], (ks / kQxStages) & 1);
            if (ks == 0 && lane == 0) ELA_TL_MARK(0);  // first stage landed
            ptx::tc_fence_after();
            if (lane == 0) {
                const uint64_t a = d0 + uint64_t((s * S::kStageBytes) >> 4);
                const uint64_t b = a + uint64_t((kQxKbp * S::kABytes) >> 4);
#pragma unroll
                for (int j = 0; j < kQxKbp; ++j) {
                    if (ks * kQxKbp + j >= p.nkb) break;
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k)
                        ptx::mma_bf16(tq, a + uint64_t((j * S::kABytes) >> 4) + uint64_t(2 * k),
                                      b + uint64_t((j * S::kBBytes) >> 4) + uint64_t(2 * k), idq, (ks | j | k) != 0);
                }
                ptx::mma_commit(&empty[s]);
            }
            __syncwarp();
        }
        if (lane == 0) ptx::mma_commit(acc_full);
        __syncwarp();
        // phase 2: q' chunks, A = Q_i (smem, written by the epilogue warps), B = W_K,i rows
        ptx::mbar_wait(q_full, 0);
        ptx::tc_fence_after();
        constexpr uint32_t idp = ptx::idesc_bf16(kBM, 128, 0, 0);
        const uint64_t aq = ptx::sdesc_sw128(ptx::smem_u32(sQ), 0, 1024);
        for (int c = 0; c < p.chunks; ++c) {
            const int bi = c & 1;
            const uint64_t bw = ptx::sdesc_sw128(ptx::smem_u32(wk_buf(bi)), 0, 1024);
            ptx::mbar_wait(&wk_full[bi], (c >> 1) & 1);
            if (c >= 2) ptx::mbar_wait(&p_empty[bi], ((c >> 1) - 1) & 1);
            ptx::tc_fence_after();
            if (lane == 0) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    ptx::mma_bf16(tp + bi * 128, aq + uint64_t(2 * k), bw + uint64_t(2 * k), idp, k != 0);
                ptx::mma_commit(&wk_empty[bi]);
                ptx::mma_commit(&p_full[bi]);
            }
            __syncwarp();
        }
    } else {
        // epilogue warps: lane quadrant qd, row = 32 qd + lane of the 128-row tile
        const uint32_t qd = warp & 3;
        const int row = int(qd) * 32 + int(lane), m = m0 + row;
        // b_Q,i: every lane needs all 64 (its row): uniform-address vector loads
        float bcol[64];
#pragma unroll
        for (int j = 0; j < 64; j += 4) {
            const float4 b4 = __ldg(reinterpret_cast<const float4*>(p.bq + z * 64 + j));
            bcol[j] = b4.x, bcol[j + 1] = b4.y, bcol[j + 2] = b4.z, bcol[j + 3] = b4.w;
        }
        ptx::mbar_wait(acc_full, 0);
        if (warp == 2 && lane == 0) ELA_TL_MARK(1);  // Q_i accumulated
        ptx::tc_fence_after();
        uint32_t v[64];
        ptx::tmem_ld32(tq + ((qd * 32) << 16), *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
        ptx::tmem_ld32(tq + ((qd * 32) << 16) + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
        ptx::tmem_ld_wait();
        // Q_i row -> bf16 -> sQ (SW128 K-major: 16-byte chunk c of row r at r*128 + ((c ^ (r & 7)) << 4))
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            uint4 o;
            o.x = pack2(__uint_as_float(v[8 * c + 0]) + bcol[8 * c + 0], __uint_as_float(v[8 * c + 1]) + bcol[8 * c + 1]);
            o.y = pack2(__uint_as_float(v[8 * c + 2]) + bcol[8 * c + 2], __uint_as_float(v[8 * c + 3]) + bcol[8 * c + 3]);
            o.z = pack2(__uint_as_float(v[8 * c + 4]) + bcol[8 * c + 4], __uint_as_float(v[8 * c + 5]) + bcol[8 * c + 5]);
            o.w = pack2(__uint_as_float(v[8 * c + 6]) + bcol[8 * c + 6], __uint_as_float(v[8 * c + 7]) + bcol[8 * c + 7]);
            *reinterpret_cast<uint4*>(sQ + uint32_t(row) * 128u + (uint32_t(c ^ (row & 7)) << 4)) = o;
        }
        ptx::fence_proxy_async_smem();  // generic-proxy writes -> the MMA's async-proxy reads
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(q_full);
        if (warp == 2 && lane == 0) ELA_TL_MARK(2);  // Q_i staged
        // phase-2 epilogue: q' chunks -> bf16 -> rows (m0 + row) * h + z
        __nv_bfloat16* dst_row = p.qp + (int64_t(m) * p.h + z) * p.d_m + col0;
        for (int c = 0; c < p.chunks; ++c) {
            const int bi = c & 1;
            ptx::mbar_wait(&p_full[bi], (c >> 1) & 1);
            ptx::tc_fence_after();
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                uint32_t r[64];
                ptx::tmem_ld32(tp + bi * 128 + half * 64 + ((qd * 32) << 16), *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
                ptx::tmem_ld32(tp + bi * 128 + half * 64 + 32 + ((qd * 32) << 16),
                               *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
                ptx::tmem_ld_wait();
                if (half == 1) {
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&p_empty[bi]);
                }
                if (m < p.M) {
                    uint4* d = reinterpret_cast<uint4*>(dst_row + c * 128 + half * 64);
#pragma unroll
                    for (int q8 = 0; q8 < 8; ++q8) {
                        uint4 w;
                        w.x = pack2(__uint_as_float(r[8 * q8 + 0]), __uint_as_float(r[8 * q8 + 1]));
                        w.y = pack2(__uint_as_float(r[8 * q8 + 2]), __uint_as_float(r[8 * q8 + 3]));
                        w.z = pack2(__uint_as_float(r[8 * q8 + 4]), __uint_as_float(r[8 * q8 + 5]));
                        w.w = pack2(__uint_as_float(r[8 * q8 + 6]), __uint_as_float(r[8 * q8 + 7]));
                        d[q8] = w;
                    }
                }
            }
        }
        if (warp == 2 && lane == 0) ELA_TL_MARK(3);  // q' stores issued
    }
    ptx::tc_fence_before();
    __syncthreads();
    ELA_TL_EXIT(kTlQexp);
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tmem);
    }
}

// Maps over an operand X[z][r][k] (r = M or N rows, k contiguous).  Loads use 4-D maps
// (64 k, r | z, z | r, k-block) whose k-block dimension has stride 128 B, so one box
// carries `kbp` k-blocks of `box_rows` rows as [kb][row][64] — KBP SWIZZLE_128B K-major
// slabs back to back.  Stores (and loads of C-shaped operands) use 3-D maps (k, r, z).
// zr_order: 1 if the coordinates are ordered (k, z, r) (keeps the r/z strides monotonic).
void dims_rz(int64_t ld, int64_t sz, int rows, int Z, uint64_t& ld_b, uint64_t& sz_b, int* zr_order) {
    ld_b = uint64_t(ld) * 2;
    sz_b = uint64_t(sz) * 2;
    if (Z == 1 || sz == 0) sz_b = ld_b * uint64_t(rows);
    *zr_order = (sz_b < ld_b && Z > 1) ? 1 : 0;
}

CUtensorMap load_map(const void* base, int64_t ld, int64_t sz, int rows, int K, int Z, uint32_t box_rows, int kbp,
                     int* zr_order) {
    uint64_t ld_b, sz_b;
    dims_rz(ld, sz, rows, Z, ld_b, sz_b, zr_order);
    const uint64_t nkb = uint64_t(K / kBK);
    if (*zr_order) {
        const uint64_t dims[4] = {uint64_t(kBK), uint64_t(Z), uint64_t(rows), nkb};
        const uint64_t strides[3] = {sz_b, ld_b, uint64_t(kBK) * 2};
        const uint32_t box[4] = {uint32_t(kBK), 1, box_rows, uint32_t(kbp)};
        return make_tmap_bf16(base, 4, dims, strides, box, 128);
    }
    const uint64_t dims[4] = {uint64_t(kBK), uint64_t(rows), uint64_t(Z), nkb};
    const uint64_t strides[3] = {ld_b, sz_b, uint64_t(kBK) * 2};
    const uint32_t box[4] = {uint32_t(kBK), box_rows, 1, uint32_t(kbp)};
    return make_tmap_bf16(base, 4, dims, strides, box, 128);
}

CUtensorMap store_map(const void* base, int64_t ld, int64_t sz, int rows, int N, int Z, uint32_t box_rows,
                      int box_cols, int* zr_order) {
    uint64_t ld_b, sz_b;
    dims_rz(ld, sz, rows, Z, ld_b, sz_b, zr_order);
    const int swz = box_cols * 2;  // 128-byte rows -> SWIZZLE_128B, 64-byte -> SWIZZLE_64B
    if (*zr_order) {
        const uint64_t dims[3] = {uint64_t(N), uint64_t(Z), uint64_t(rows)};
        const uint64_t strides[2] = {sz_b, ld_b};
        const uint32_t box[3] = {uint32_t(box_cols), 1, box_rows};
        return make_tmap_bf16(base, 3, dims, strides, box, swz);
    }
    const uint64_t dims[3] = {uint64_t(N), uint64_t(rows), uint64_t(Z)};
    const uint64_t strides[2] = {ld_b, sz_b};
    const uint32_t box[3] = {uint32_t(box_cols), box_rows, 1};
    return make_tmap_bf16(base, 3, dims, strides, box, swz);
}

int num_sms() {
    static int n = [] {
        int dev = 0, v = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return n;
}

template <int BN, int MT, int KBP, bool BIAS, bool SCALE>
void launch_cfg(const GemmArgs& g, cudaStream_t st) {
    using S = GemmSmem<BN, MT, KBP>;
    GemmParams p{};
    p.M = g.M, p.N = g.N, p.K = g.K, p.Z = g.Z, p.alpha = g.alpha, p.bias = g.bias, p.sbz = g.sbz;
    p.tiles_m = int(ceil_div(g.M, int64_t(kBM) * MT));
    p.tiles_n = int(ceil_div(g.N, BN));
    p.a_bcast = (g.Z > 1 && g.sAz == 0) ? 1 : 0;
    p.pdl = pdl_enabled() ? 1 : 0;
    // write-bound q' expansion (BN = 256): TMA stores; the others: coalesced st.global
    p.direct = g_gemm_epilogue_tma < 0 ? (BN == 256 ? 0 : 1) : (g_gemm_epilogue_tma ? 0 : 1);
    p.C = static_cast<__nv_bfloat16*>(g.C), p.ldc = g.ldc, p.sCz = g.sCz;
    p.trace = g_gemm_trace;
    // weights: evict-last keeps a weight tile in L2 while every M-block of this GEMM reads
    // it; ELATTN_GEMM_W_POLICY=normal|first for L2 experiments (H residency at small B)
    static const uint64_t w_pol = [] {
        const char* e = getenv("ELATTN_GEMM_W_POLICY");
        const std::string v = e ? e : "";
        return v == "normal" ? ptx::kEvictNormal : v == "first" ? ptx::kEvictFirst : ptx::kEvictLast;
    }();
    p.b_pol = w_pol;
    // output: evict-last when the next kernel re-reads it while a large stream passes through
    // L2 (the q' expansion, read by the decode while H streams evict-first)
    static const uint64_t c_keep = [] {
        const char* e = getenv("ELATTN_GEMM_C_POLICY");
        const std::string v = e ? e : "";
        return v == "normal" ? ptx::kEvictNormal : ptx::kEvictLast;
    }();
    p.c_pol = g.c_keep ? c_keep : ptx::kEvictNormal;
    {
        const int num_ks = int(ceil_div(g.K / kBK, KBP));
        p.b_pre = (g.b_static && p.pdl) ? (num_ks < S::kStages ? num_ks : S::kStages) : 0;
    }
    CUtensorMap ta = load_map(g.A, g.lda, g.sAz, g.M, g.K, p.a_bcast ? 1 : g.Z, kBM, KBP, &p.a_zm);
    CUtensorMap tb = load_map(g.B, g.ldb, g.sBz, g.N, g.K, g.Z, BN, KBP, &p.b_zm);
    CUtensorMap tc = store_map(g.C, g.ldc, g.sCz, g.M, g.N, g.Z, kBM, S::kPiece, &p.c_zm);
    auto kern = tc_gemm_kernel<BN, MT, KBP, BIAS, SCALE>;
    constexpr uint32_t smem = S::kTotal;
    ELA_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const int tiles = p.Z * p.tiles_m * p.tiles_n;
    const int grid = tiles < num_sms() ? tiles : num_sms();
    // a stage always expects KBP full k-blocks: a short last stage (K / 64 not a multiple
    // of KBP) is completed by the zero-filled out-of-range part of the box
    launch_ex(kern, dim3(grid), dim3(kThreads), smem, st, 1, ta, tb, tc, p);
    ELA_CHECK_LAUNCH();
}

template <int BN, int MT, int KBP>
void launch_variant(const GemmArgs& g, cudaStream_t st) {
    const bool bias = g.bias != nullptr, scale = g.alpha != 1.f;
    if (bias && scale) return launch_cfg<BN, MT, KBP, true, true>(g, st);
    if (bias) return launch_cfg<BN, MT, KBP, true, false>(g, st);
    if (scale) return launch_cfg<BN, MT, KBP, false, true>(g, st);
    return launch_cfg<BN, MT, KBP, false, false>(g, st);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

struct Cfg {
    int bn, mt, kbp;
};

// Block shape per GEMM (B200, 148 SMs):
//   * N <= 64 (per-head V projection, N = d_k): 128 x 64 tiles, two m-subtiles per CTA
//     sharing the weight slice beyond two waves of single tiles;
//   * K <= 128 (q' expansion, write-bound): 128 x 256 tiles (128 x 128 for small M), one k-step;
//   * otherwise (Y.W_Q, V.W_O): 128 x 128 tiles;
// with two k-blocks per TMA box whenever K allows.
Cfg choose(const GemmArgs& g) {
    Cfg c{128, 1, 2};
    if (g.N <= 64) {
        c = {64, 1, 2};
        const int64_t tiles = ceil_div(g.M, kBM) * g.Z;
        // two m-subtiles (halving the weight traffic) only beyond two waves of single tiles:
        // up to two waves, one subtile per CTA keeps all 148 SMs streaming A (the decode's C,
        // read from DRAM inside the step): B = 296 / 320 step -0.5% (80 -> 148 CTAs)
        if (g.K >= 256 && tiles > 2 * num_sms()) c.mt = 2;
    } else if (g.K <= 128) {
        // write-bound q' expansion: 256-wide tiles, unless that leaves half the SMs idle
        // (small batches: 128-wide, measured 3.4 vs 4.3 us at B = 32, tools/time_gemms.py)
        const int64_t tiles256 = ceil_div(g.M, kBM) * ceil_div(g.N, 256) * g.Z;
        c = {(g.N >= 256 && 2 * tiles256 >= num_sms()) ? 256 : 128, 1, 1};
    }
    if (g.K / kBK < 2) c.kbp = 1;
    if (g_gemm_force_bn) c.bn = g_gemm_force_bn;
    if (g_gemm_force_mt) c.mt = g_gemm_force_mt;
    if (g_gemm_force_kbp) c.kbp = g_gemm_force_kbp;
    if (c.bn > 64 && g.N <= 64) c.bn = 64;
    return c;
}

// split-K for small M: cluster size SK (2, 4, 8), 0 when the tile grid already fills the GPU

int choose_splitk(const GemmArgs& g) {
    const int nkb = g.K / kBK;
    const int64_t tiles = ceil_div(g.M, kBM) * ceil_div(g.N, kSkBN) * g.Z;
    auto ok = [&](int sk) { return nkb % sk == 0 && nkb / sk <= int(SkSmem<2>::kMaxKbp) && (kSkBN / sk) % 8 == 0; };
    if (g_gemm_force_splitk >= 0) return (g_gemm_force_splitk > 1 && ok(g_gemm_force_splitk)) ? g_gemm_force_splitk : 0;
    static const int env = [] {
        const char* e = getenv("ELATTN_GEMM_SPLITK");
        return e ? atoi(e) : -1;
    }();
    if (env >= 0) return (env > 1 && ok(env)) ? env : 0;
    if (nkb < 4 || 2 * tiles > num_sms()) return 0;
    // one wave of co-resident clusters (tools/probes/cluster_occupancy_probe.cu on B200:
    // 74 clusters of 2, 33 of 4, 15 of 8 for a one-CTA-per-SM kernel)
    const int sms = num_sms();
    const int64_t max_cl[3] = {sms / 2, (sms * 33) / 148, (sms * 15) / 148};
    const int sks[3] = {2, 4, 8};
    // the widest split whose clusters are all co-resident in one wave, at most ~64 CTAs —
    // or up to one CTA per SM when every row tile is full (since the bulk-DSMEM exchange,
    // SK = 4 on 128 CTAs beats pairs at B = 64, step -1%, but not at B = 48, whose second
    // row tile is half empty: +0.7%; profiles/r02c_splitk_factor_sweep*.txt)
    const bool full_rows = g.M % kBM == 0;
    for (int i = 2; i >= 0; --i)
        if (ok(sks[i]) && tiles <= max_cl[i] &&
            (tiles * sks[i] <= 64 || sks[i] == 2 || (full_rows && tiles * sks[i] <= sms)))
            return sks[i];
    return 0;
}

template <int SK, bool BIAS, bool SCALE>
void launch_splitk_cfg(const GemmArgs& g, cudaStream_t st) {
    using S = SkSmem<SK>;
    SkParams p{};
    p.M = g.M, p.N = g.N, p.K = g.K, p.Z = g.Z;
    p.tiles_m = int(ceil_div(g.M, kBM));
    p.tiles_n = int(ceil_div(g.N, kSkBN));
    p.kbp = g.K / kBK / SK;
    p.a_bcast = (g.Z > 1 && g.sAz == 0) ? 1 : 0;
    p.pdl = pdl_enabled() ? 1 : 0;
    p.b_static = g.b_static;
    p.alpha = g.alpha, p.bias = g.bias, p.sbz = g.sbz;
    p.C = static_cast<__nv_bfloat16*>(g.C), p.ldc = g.ldc, p.sCz = g.sCz;
    CUtensorMap ta = load_map(g.A, g.lda, g.sAz, g.M, g.K, p.a_bcast ? 1 : g.Z, kBM, p.kbp, &p.a_zm);
    CUtensorMap tb = load_map(g.B, g.ldb, g.sBz, g.N, g.K, g.Z, kSkBN, p.kbp, &p.b_zm);
    auto kern = tc_gemm_splitk_kernel<SK, BIAS, SCALE>;
    ELA_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(S::kTotal)));
    const int clusters = p.Z * p.tiles_m * p.tiles_n;
    launch_ex(kern, dim3(clusters * SK), dim3(kSkThreads), S::kTotal, st, SK, ta, tb, p);
    ELA_CHECK_LAUNCH();
}

template <int SK>
void launch_splitk(const GemmArgs& g, cudaStream_t st) {
    const bool bias = g.bias != nullptr, scale = g.alpha != 1.f;
    if (bias && scale) return launch_splitk_cfg<SK, true, true>(g, st);
    if (bias) return launch_splitk_cfg<SK, true, false>(g, st);
    if (scale) return launch_splitk_cfg<SK, false, true>(g, st);
    return launch_splitk_cfg<SK, false, false>(g, st);
}

// Rows for which the fused query expansion is used automatically: M <= 64 and
// 128 < M <= qexp_max_rows() (default 256; ELATTN_QEXP_ROWS overrides the bound).  Measured
// in the 12-layer step (profiles/r02c_qexp_threshold.jsonl): B = 8 / 16 -1% / -1%, B = 48 /
// 64 (two row tiles) -3% / -1.8%; at 65..128 rows (B = 24 / 32, one row tile, 64 CTAs) the
// split-K Q GEMM + q' GEMM stay 0.4-0.5% ahead.
int qexp_max_rows() {
    static const int v = [] {
        const char* e = getenv("ELATTN_QEXP_ROWS");
        return e ? atoi(e) : 256;
    }();
    return v;
}

// fused query expansion for small batches (see tc_qexp_kernel); false = not applicable
bool launch_qexp_fused(const void* Y, int M, const void* WqT, const float* bq, const void* Wk, void* qp, int h,
                       int d_m, int d_k, cudaStream_t st) {
    static const int env = [] {
        const char* e = getenv("ELATTN_QEXP_FUSED");
        return e ? atoi(e) : -1;
    }();
    if (env == 0 || g_qexp_fused == 0) return false;
    const int items = int(ceil_div(M, kBM)) * h;
    if (d_k != 64 || d_m % 512 != 0 || 4 * items > 2 * num_sms()) return false;
    if (g_qexp_fused < 0 && env < 0 && (M > qexp_max_rows() || (M > 64 && M <= 128))) return false;
    if (bq == nullptr || !aligned16(Y) || !aligned16(WqT) || !aligned16(Wk) || !aligned16(qp) || !aligned16(bq)) return false;
    QxParams p{};
    p.M = M, p.d_m = d_m, p.h = h, p.nkb = d_m / kBK, p.nks = int(ceil_div(d_m / kBK, kQxKbp)), p.chunks = d_m / 4 / 128;
    p.pdl = pdl_enabled() ? 1 : 0;
    p.bq = bq;
    p.qp = static_cast<__nv_bfloat16*>(qp);
    int zr = 0;
    // Y [M][d_m]: 4-D map (64 k, rows, 1, k-block); W_Q^T [h*64][d_m] likewise; W_K [h][d_m][64]: 3-D (k, d, head)
    CUtensorMap ty = load_map(Y, d_m, 0, M, d_m, 1, kBM, kQxKbp, &zr);
    CUtensorMap twq = load_map(WqT, d_m, 0, h * 64, d_m, 1, 64, kQxKbp, &zr);
    const uint64_t kd[3] = {uint64_t(d_k), uint64_t(d_m), uint64_t(h)};
    const uint64_t ks[2] = {uint64_t(d_k) * 2, uint64_t(d_m) * d_k * 2};
    const uint32_t kbox[3] = {64, 128, 1};
    CUtensorMap twk = make_tmap_bf16(Wk, 3, kd, ks, kbox, 128);
    ELA_CHECK_CUDA(cudaFuncSetAttribute(tc_qexp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(QxSmem::kTotal)));
    launch_ex(tc_qexp_kernel, dim3(items * 4), dim3(kQxThreads), QxSmem::kTotal, st, 1, ty, twq, twk, p);
    ELA_CHECK_LAUNCH();
    return true;
}

}  // namespace

bool tc_qexp_fused(const void* Y, int M, const void* WqT, const float* bq, const void* Wk, void* qp, int h, int d_m,
                   int d_k, cudaStream_t st) {
    return launch_qexp_fused(Y, M, WqT, bq, Wk, qp, h, d_m, d_k, st);
}

bool tc_gemm_supported(const GemmArgs& g) {
    return g.K % kBK == 0 && g.K > 0 && g.N % 16 == 0 && g.M > 0 && g.lda % 8 == 0 && g.ldb % 8 == 0 &&
           g.ldc % 8 == 0 && g.sAz % 8 == 0 && g.sBz % 8 == 0 && g.sCz % 8 == 0 && aligned16(g.A) &&
           aligned16(g.B) && aligned16(g.C);
}

void launch_tc_gemm(const GemmArgs& g, cudaStream_t st) {
    if (!g_gemm_force_bn && !g_gemm_force_mt && !g_gemm_force_kbp) {
        switch (choose_splitk(g)) {
            case 8: return launch_splitk<8>(g, st);
            case 4: return launch_splitk<4>(g, st);
            case 2: return launch_splitk<2>(g, st);
            default: break;
        }
    }
    const Cfg c = choose(g);
    const int key = c.bn * 100 + c.mt * 10 + c.kbp;
    switch (key) {
        case 6411: return launch_variant<64, 1, 1>(g, st);
        case 6412: return launch_variant<64, 1, 2>(g, st);
        case 6421: return launch_variant<64, 2, 1>(g, st);
        case 6422: return launch_variant<64, 2, 2>(g, st);
        case 12811: return launch_variant<128, 1, 1>(g, st);
        case 12812: return launch_variant<128, 1, 2>(g, st);
        case 12821: return launch_variant<128, 2, 1>(g, st);
        case 12822: return launch_variant<128, 2, 2>(g, st);
        case 25611: return launch_variant<256, 1, 1>(g, st);
        case 25612: return launch_variant<256, 1, 2>(g, st);
        default:
            throw Status{ELATTN_ERR_UNSUPPORTED, "tc_gemm: no instantiation for BN " + std::to_string(c.bn) +
                                                     " MT " + std::to_string(c.mt) + " KBP " + std::to_string(c.kbp)};
    }
}

ELA_TL_SETTER(tl_set_gemm)

}  // namespace elattn_gpu
