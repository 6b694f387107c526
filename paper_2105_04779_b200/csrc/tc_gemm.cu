// tc_gemm.cu — persistent tcgen05 GEMM for the projection stages of the bf16 path.
//
//   C[z][m][n] = alpha * sum_k A[z][m][k] * B[z][n][k] + bias[z][n]     (bf16 in/out)
//
// Replaces the reference's CPU matmuls of query expansion (attention.hpp:205-206:
// q.Wq_i + bq_i, Q_i.Wk_i^T) and of the output projection (:286, :221-231:
// ctx.Wv_i + bv_i, then .Wo + bo).
//
// Persistent, warp-specialised: one CTA per SM walks 128 x BN output tiles
// (n fastest, so consecutive tiles reuse the A block from L2).
//   warp 0      TMA producer: 128x64 / BNx64 bf16 K-slices (SWIZZLE_128B) through an
//               mbarrier ring;
//   warp 1      MMA issuer (tcgen05.mma M=128 N=BN K=16, fp32 accumulator in TMEM,
//               double-buffered so the epilogue of tile t overlaps the MMAs of t+1);
//   warps 2..9  epilogue, two warps per TMEM lane quadrant (column halves):
//               tcgen05.ld -> alpha/bias -> bf16 -> SWIZZLE_128B smem stage (double
//               buffered) -> TMA tensor store (3-D maps, so head-strided outputs such
//               as q' rows r*h + i are written directly).  The write-bound shapes
//               (q' = Q_i.Wk_i^T: K = 64, 42 MB out at B = 320) live in this epilogue.
#include "common.cuh"
#include "kernels.h"
#include "ptx_sm100.cuh"
#include "tmap.h"

namespace elattn_gpu {

namespace {

constexpr int kBM = 128, kBK = 64;
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;

template <int BN>
struct GemmSmem {
    static constexpr uint32_t kABytes = kBM * kBK * 2;
    static constexpr uint32_t kBBytes = BN * kBK * 2;
    static constexpr uint32_t kStageBytes = kABytes + kBBytes;
    // epilogue: every warp stages its own 32 rows x BN/2 columns as 32-row x 64-column
    // SWIZZLE_128B boxes (4 KB each) and stores them itself, double buffered
    static constexpr int kBoxCols = BN / 2 < 64 ? BN / 2 : 64;  // 64 (SW128) or 32 (SW64)
    static constexpr uint32_t kWarpBox = 32 * kBoxCols * 2;
    static constexpr uint32_t kWarpStage = (BN / 2) / kBoxCols * kWarpBox;
    static constexpr int kOutStages = 3;
    static constexpr uint32_t kOutBytes = kEpiWarps * kOutStages * kWarpStage;
    static constexpr uint32_t kFixed = kOutBytes + 256 + 1024;
    static constexpr int kStagesFit = int((232448u - kFixed) / kStageBytes);
    static constexpr int kStages = kStagesFit < 8 ? kStagesFit : 8;
    static constexpr uint32_t kOutOff = kStages * kStageBytes;
    static constexpr uint32_t kBarOff = kOutOff + kOutBytes;
    static constexpr uint32_t kTotal = kBarOff + 256 + 1024;  // + barriers + alignment slack
    static_assert(kTotal <= 232448, "smem");
};

struct GemmParams {
    int M, N, K, Z;
    int tiles_m, tiles_n;
    float alpha;
    const float* bias;
    int64_t sbz;
    int a_zm, b_zm, c_zm;  // 1: tensor map coordinate order is (k, z, m) instead of (k, m, z)
    int a_bcast;  // A shared by every z (sAz == 0): load it with z = 0
};


__device__ __forceinline__ uint32_t pack2(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
}

template <int BN, bool BIAS, bool SCALE>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, GemmParams p) {
    using S = GemmSmem<BN>;
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
    constexpr uint32_t kTmemCols = 2 * BN < 32 ? 32 : 2 * BN;

    const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
    const int num_k = p.K / kBK;
    const int num_tiles = p.Z * p.tiles_m * p.tiles_n;
    // z (head) fastest: the CTAs running concurrently touch the SAME rows r of the
    // head-interleaved layouts (q' / C rows r*h + i), so their 128-byte row pieces land
    // in the same DRAM pages instead of 32 KB apart
    auto tile_coords = [&](int t, int& z, int& m0, int& n0) {
        z = t % p.Z;
        const int r = t / p.Z;
        m0 = (r / p.tiles_n) * kBM;
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
        ptx::tmem_alloc<kTmemCols>(tmem_slot);
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---- TMA producer
        if (ptx::elect_one()) {
            int it = 0;
            for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
                int z, m0, n0;
                tile_coords(t, z, m0, n0);
                for (int kb = 0; kb < num_k; ++kb, ++it) {
                    const int s = it % kStages;
                    ptx::mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
                    uint8_t* a = smem + s * S::kStageBytes;
                    uint8_t* b = a + S::kABytes;
                    ptx::mbar_arrive_expect_tx(&full[s], S::kStageBytes);
                    const int za = p.a_bcast ? 0 : z;
                    if (p.a_zm)
                        ptx::tma_load_3d(a, &tmA, &full[s], kb * kBK, za, m0, ptx::kEvictNormal);
                    else
                        ptx::tma_load_3d(a, &tmA, &full[s], kb * kBK, m0, za, ptx::kEvictNormal);
                    if (p.b_zm)
                        ptx::tma_load_3d(b, &tmB, &full[s], kb * kBK, z, n0, ptx::kEvictLast);
                    else
                        ptx::tma_load_3d(b, &tmB, &full[s], kb * kBK, n0, z, ptx::kEvictLast);
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
            const uint32_t d = tmem + ab * BN;
            for (int kb = 0; kb < num_k; ++kb, ++it) {
                const int s = it % kStages;
                ptx::mbar_wait(&full[s], (it / kStages) & 1);
                ptx::tc_fence_after();
                if (lane == 0) {
                    const uint64_t a = d0 + uint64_t((s * S::kStageBytes) >> 4);
                    const uint64_t b = a + uint64_t(S::kABytes >> 4);
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k)
                        ptx::mma_bf16(d, a + uint64_t(2 * k), b + uint64_t(2 * k), idesc, (kb | k) != 0);
                    ptx::mma_commit(&empty[s]);
                }
                __syncwarp();
            }
            if (lane == 0) ptx::mma_commit(&acc_full[ab]);
            __syncwarp();
        }
    } else {
        // ---- epilogue warps 2..9: quadrant qd = warp % 4 (TMEM lanes / tile rows
        // 32 qd..), column half ch = (warp - 2) / 4 (tile columns ch*BN/2 ..).  Each warp
        // is independent: TMEM -> registers -> its own SWIZZLE_128B stage -> its own TMA
        // store (boxes of 32 rows x 64 columns); no CTA-wide barrier in the tile loop.
        const uint32_t qd = warp & 3, ch = (warp - 2) >> 2;
        constexpr int kHalf = BN / 2;
        uint8_t* my_stage = out_stage + (warp - 2) * S::kOutStages * S::kWarpStage;
        int local = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++local) {
            int z, m0, n0;
            tile_coords(t, z, m0, n0);
            const int ab = local & 1;
            uint8_t* stage = my_stage + (local % S::kOutStages) * S::kWarpStage;
            ptx::mbar_wait(&acc_full[ab], (local >> 1) & 1);
            ptx::tc_fence_after();
            const uint32_t t_row = tmem + ((qd * 32) << 16) + ab * BN + ch * kHalf;
            uint32_t rr[kHalf];  // this warp's 32 rows x kHalf columns, one TMEM round trip
#pragma unroll
            for (int c0 = 0; c0 < kHalf; c0 += 32) ptx::tmem_ld32(t_row + c0, *reinterpret_cast<uint32_t(*)[32]>(&rr[c0]));
            ptx::tmem_ld_wait();
            // this warp's part of the accumulator is read: the MMA warp may reuse it
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                ptx::mbar_arrive(&acc_empty[ab]);
                ptx::bulk_wait_group_read<S::kOutStages - 1>();  // this stage's previous store has read it
            }
            __syncwarp();
            // bias of this warp's columns: lane l holds column c0 + l of each 32-column
            // chunk, broadcast with shuffles (no per-element loads)
            float bcol[kHalf / 32];
            if constexpr (BIAS) {
#pragma unroll
                for (int c = 0; c < kHalf / 32; ++c) {
                    const int n = n0 + int(ch) * kHalf + 32 * c + int(lane);
                    bcol[c] = n < p.N ? __ldg(p.bias + z * p.sbz + n) : 0.f;
                }
            }
#pragma unroll
            for (int c0 = 0; c0 < kHalf; c0 += 32) {
                const uint32_t* r = rr + c0;
                uint32_t packed[16];
#pragma unroll
                for (int j = 0; j < 32; j += 2) {
                    float v0 = __uint_as_float(r[j]), v1 = __uint_as_float(r[j + 1]);
                    if constexpr (SCALE) v0 *= p.alpha, v1 *= p.alpha;
                    if constexpr (BIAS) {
                        v0 += __shfl_sync(0xffffffffu, bcol[c0 / 32], j);
                        v1 += __shfl_sync(0xffffffffu, bcol[c0 / 32], j + 1);
                    }
                    packed[j / 2] = pack2(v0, v1);
                }
                // 32-row box of kBoxCols columns: SWIZZLE_128B (16-byte chunk c of row l at
                // c ^ (l & 7)) for 64 columns, SWIZZLE_64B (c ^ ((l >> 1) & 3)) for 32
                constexpr int kBoxCols = S::kBoxCols;
                uint8_t* box = stage + (c0 / kBoxCols) * S::kWarpBox + lane * (kBoxCols * 2);
                const int cbase = (c0 % kBoxCols) >> 3;
                const int sw = kBoxCols == 64 ? int(lane & 7) : int((lane >> 1) & 3);
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    *reinterpret_cast<uint4*>(box + (((cbase + q) ^ sw) << 4)) =
                        make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
            }
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
#pragma unroll
                for (int bx = 0; bx < kHalf / S::kBoxCols; ++bx) {
                    const int c0 = n0 + int(ch) * kHalf + S::kBoxCols * bx;
                    if (c0 >= p.N) break;
                    const int r0 = m0 + int(qd) * 32;
                    if (p.c_zm)
                        ptx::tma_store_3d(&tmC, stage + bx * S::kWarpBox, c0, z, r0);
                    else
                        ptx::tma_store_3d(&tmC, stage + bx * S::kWarpBox, c0, r0, z);
                }
                ptx::bulk_commit_group();
            }
        }
        if (lane == 0) ptx::bulk_wait_group<0>();
        __syncwarp();
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<kTmemCols>(tmem);
    }
}

// 3-D map over an operand X[z][r][k] (r = M or N rows, k contiguous):
// returns the map and whether coordinates are ordered (k, z, r).
CUtensorMap operand_map(const void* base, int64_t ld, int64_t sz, int rows, int K, int Z, uint32_t box_rows,
                        int* zr_order, int box_k = kBK) {
    const int swz = box_k * 2;  // 128-byte rows -> SWIZZLE_128B, 64-byte -> SWIZZLE_64B
    const uint64_t ld_b = uint64_t(ld) * 2;
    uint64_t sz_b = uint64_t(sz) * 2;
    if (Z == 1 || sz == 0) sz_b = ld_b * uint64_t(rows);
    if (sz_b < ld_b && Z > 1) {  // keep strides monotonic: dims (k, z, r)
        const uint64_t dims[3] = {uint64_t(K), uint64_t(Z), uint64_t(rows)};
        const uint64_t strides[2] = {sz_b, ld_b};
        const uint32_t box[3] = {uint32_t(box_k), 1, box_rows};
        *zr_order = 1;
        return make_tmap_bf16(base, 3, dims, strides, box, swz);
    }
    const uint64_t dims[3] = {uint64_t(K), uint64_t(rows), uint64_t(Z)};
    const uint64_t strides[2] = {ld_b, sz_b};
    const uint32_t box[3] = {uint32_t(box_k), box_rows, 1};
    *zr_order = 0;
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

template <int BN, bool BIAS, bool SCALE>
void launch_bn(const GemmArgs& g, cudaStream_t st) {
    GemmParams p{};
    p.M = g.M, p.N = g.N, p.K = g.K, p.Z = g.Z, p.alpha = g.alpha, p.bias = g.bias, p.sbz = g.sbz;
    p.tiles_m = int(ceil_div(g.M, kBM));
    p.tiles_n = int(ceil_div(g.N, BN));
    p.a_bcast = (g.Z > 1 && g.sAz == 0) ? 1 : 0;
    CUtensorMap ta = operand_map(g.A, g.lda, g.sAz, g.M, g.K, p.a_bcast ? 1 : g.Z, kBM, &p.a_zm);
    CUtensorMap tb = operand_map(g.B, g.ldb, g.sBz, g.N, g.K, g.Z, BN, &p.b_zm);
    // output C[z][m][n]: boxes of 32 rows x kBoxCols columns (one epilogue warp's piece),
    // clipped at M / N
    CUtensorMap tc = operand_map(g.C, g.ldc, g.sCz, g.M, g.N, g.Z, 32, &p.c_zm, GemmSmem<BN>::kBoxCols);
    auto kern = tc_gemm_kernel<BN, BIAS, SCALE>;
    constexpr uint32_t smem = GemmSmem<BN>::kTotal;
    ELA_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const int tiles = p.Z * p.tiles_m * p.tiles_n;
    const int grid = tiles < num_sms() ? tiles : num_sms();
    kern<<<grid, kThreads, smem, st>>>(ta, tb, tc, p);
    ELA_CHECK_LAUNCH();
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

bool tc_gemm_supported(const GemmArgs& g) {
    return g.K % kBK == 0 && g.K > 0 && g.N % 16 == 0 && g.M > 0 && g.lda % 8 == 0 && g.ldb % 8 == 0 &&
           g.ldc % 8 == 0 && g.sAz % 8 == 0 && g.sBz % 8 == 0 && g.sCz % 8 == 0 && aligned16(g.A) &&
           aligned16(g.B) && aligned16(g.C);
}

template <int BN>
void launch_variant(const GemmArgs& g, cudaStream_t st) {
    const bool bias = g.bias != nullptr, scale = g.alpha != 1.f;
    if (bias && scale) return launch_bn<BN, true, true>(g, st);
    if (bias) return launch_bn<BN, true, false>(g, st);
    if (scale) return launch_bn<BN, false, true>(g, st);
    return launch_bn<BN, false, false>(g, st);
}

void launch_tc_gemm(const GemmArgs& g, cudaStream_t st) {
    if (g.N <= 64)
        launch_variant<64>(g, st);
    else
        launch_variant<128>(g, st);
}

}  // namespace elattn_gpu
