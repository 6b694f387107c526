// tc_gemm.cu — tcgen05 GEMM for the projection stages of the bf16 path.
//
//   C[z][m][n] = alpha * sum_k A[z][m][k] * B[z][n][k] + bias[z][n]     (bf16 in/out)
//
// Replaces the reference's CPU matmuls of query expansion (attention.hpp:205-206:
// q.Wq_i + bq_i, Q_i.Wk_i^T) and of the output projection (:286, :221-231:
// ctx.Wv_i + bv_i, then .Wo + bo).  One 128 x BN output tile per CTA:
// a TMA producer (warp 0) streams 128x64 / BNx64 bf16 K-slices (SWIZZLE_128B)
// through a 4-stage mbarrier ring, a single thread (warp 1) issues
// tcgen05.mma (M=128, N=BN, K=16) into a TMEM fp32 accumulator, and all four
// warps run the epilogue (tcgen05.ld -> alpha/bias -> bf16 -> st.global).
#include "common.cuh"
#include "kernels.h"
#include "ptx_sm100.cuh"
#include "tmap.h"

namespace elattn_gpu {

namespace {

constexpr int kBM = 128, kBK = 64, kStages = 4;

template <int BN>
struct GemmSmem {
    static constexpr uint32_t kABytes = kBM * kBK * 2;
    static constexpr uint32_t kBBytes = BN * kBK * 2;
    static constexpr uint32_t kStageBytes = kABytes + kBBytes;
    static constexpr uint32_t kBarOff = kStages * kStageBytes;
    static constexpr uint32_t kTotal = kBarOff + 256 + 1024;  // + barriers + alignment slack
};

struct GemmParams {
    int M, N, K;
    float alpha;
    const float* bias;
    int64_t sbz;
    __nv_bfloat16* C;
    int64_t ldc, sCz;
    int a_zm, b_zm;  // 1: tensor map coordinate order is (k, z, m) instead of (k, m, z)
};

template <int BN>
__global__ void __launch_bounds__(128, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmParams p) {
    using S = GemmSmem<BN>;
    extern __shared__ uint8_t smem_raw[];
    // 1024-B alignment for SWIZZLE_128B, by offsetting the __shared__ array itself so
    // the compiler keeps the shared address space (LDS/STS, not generic LD/ST)
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kBarOff);
    uint64_t* empty = full + kStages;
    uint64_t* accum_full = empty + kStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum_full + 1);
    constexpr uint32_t kTmemCols = BN < 32 ? 32 : BN;

    const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
    const int m0 = blockIdx.y * kBM, n0 = blockIdx.x * BN, z = blockIdx.z;
    const int num_k = p.K / kBK;

    if (warp == 0) {
        if (ptx::elect_one()) {
            ptx::prefetch_tmap(&tmA);
            ptx::prefetch_tmap(&tmB);
            for (int s = 0; s < kStages; ++s) {
                ptx::mbar_init(&full[s], 1);
                ptx::mbar_init(&empty[s], 1);
            }
            ptx::mbar_init(accum_full, 1);
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
        if (ptx::elect_one()) {  // ---- TMA producer
            for (int kb = 0; kb < num_k; ++kb) {
                const int s = kb % kStages;
                const uint32_t ph = (kb / kStages) & 1;
                ptx::mbar_wait(&empty[s], ph ^ 1);
                uint8_t* a = smem + s * S::kStageBytes;
                uint8_t* b = a + S::kABytes;
                ptx::mbar_arrive_expect_tx(&full[s], S::kStageBytes);
                if (p.a_zm)
                    ptx::tma_load_3d(a, &tmA, &full[s], kb * kBK, z, m0, ptx::kEvictNormal);
                else
                    ptx::tma_load_3d(a, &tmA, &full[s], kb * kBK, m0, z, ptx::kEvictNormal);
                if (p.b_zm)
                    ptx::tma_load_3d(b, &tmB, &full[s], kb * kBK, z, n0, ptx::kEvictLast);
                else
                    ptx::tma_load_3d(b, &tmB, &full[s], kb * kBK, n0, z, ptx::kEvictLast);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (ptx::elect_one()) {  // ---- MMA issuer
            constexpr uint32_t idesc = ptx::idesc_bf16(kBM, BN, 0, 0);
            for (int kb = 0; kb < num_k; ++kb) {
                const int s = kb % kStages;
                const uint32_t ph = (kb / kStages) & 1;
                ptx::mbar_wait(&full[s], ph);
                ptx::tc_fence_after();
                const uint32_t a = ptx::smem_u32(smem + s * S::kStageBytes);
                const uint32_t b = a + S::kABytes;
#pragma unroll
                for (int k = 0; k < kBK / 16; ++k)
                    ptx::mma_bf16(tmem, ptx::sdesc_sw128(a + 32 * k, 0, 1024), ptx::sdesc_sw128(b + 32 * k, 0, 1024),
                                  idesc, (kb | k) != 0);
                ptx::mma_commit(&empty[s]);
            }
            ptx::mma_commit(accum_full);
        }
        __syncwarp();
    }

    // ---- epilogue: TMEM -> registers (thread = row) -> alpha/bias -> bf16 -> smem
    // staging tile (the drained A/B stages) -> coalesced 16-byte global stores.
    ptx::mbar_wait(accum_full, 0);
    ptx::tc_fence_after();
    constexpr int kPitch = BN * 2 + 16;  // bytes per staged row (+16: spread banks)
    static_assert(kBM * kPitch <= kStages * S::kStageBytes, "staging tile fits in the pipeline buffers");
    const int r_local = int(warp) * 32 + int(lane);
    const uint32_t t_row = tmem + ((warp * 32) << 16);
    const float* bias = p.bias ? p.bias + z * p.sbz : nullptr;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t r[16];
        ptx::tmem_ld16(t_row + c0, r);
        ptx::tmem_ld_wait();
        const int n = n0 + c0;
        uint32_t packed[8];
#pragma unroll
        for (int j = 0; j < 16; j += 2) {
            float v0 = __uint_as_float(r[j]) * p.alpha, v1 = __uint_as_float(r[j + 1]) * p.alpha;
            if (bias) {
                v0 += (n + j < p.N) ? bias[n + j] : 0.f;
                v1 += (n + j + 1 < p.N) ? bias[n + j + 1] : 0.f;
            }
            __nv_bfloat162 h2 = __floats2bfloat162_rn(v0, v1);
            packed[j / 2] = *reinterpret_cast<uint32_t*>(&h2);
        }
        uint8_t* dst = smem + r_local * kPitch + c0 * 2;
        *reinterpret_cast<uint4*>(dst) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
        *reinterpret_cast<uint4*>(dst + 16) = make_uint4(packed[4], packed[5], packed[6], packed[7]);
    }
    __syncthreads();
    constexpr int kVecPerRow = BN / 8;  // 16-byte vectors per output row
    const bool full_n = (n0 + BN <= p.N) && (p.N % 8 == 0);
#pragma unroll 4
    for (int idx = int(threadIdx.x); idx < kBM * kVecPerRow; idx += 128) {
        const int rr = idx / kVecPerRow, cv = idx % kVecPerRow;
        const int row = m0 + rr, n = n0 + cv * 8;
        if (row >= p.M) continue;
        __nv_bfloat16* Crow = p.C + z * p.sCz + int64_t(row) * p.ldc;
        const uint8_t* src = smem + rr * kPitch + cv * 16;
        if (full_n || n + 8 <= p.N) {
            *reinterpret_cast<uint4*>(Crow + n) = *reinterpret_cast<const uint4*>(src);
        } else {
            for (int j = 0; j < 8 && n + j < p.N; ++j) Crow[n + j] = reinterpret_cast<const __nv_bfloat16*>(src)[j];
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) ptx::tmem_dealloc<kTmemCols>(tmem);
}

// 3-D map over an operand X[z][r][k] (r = M or N rows, k contiguous):
// returns the map and whether coordinates are ordered (k, z, r).
CUtensorMap operand_map(const void* base, int64_t ld, int64_t sz, int rows, int K, int Z, uint32_t box_rows,
                        int* zr_order) {
    const uint64_t ld_b = uint64_t(ld) * 2;
    uint64_t sz_b = uint64_t(sz) * 2;
    if (Z == 1 || sz == 0) sz_b = ld_b * uint64_t(rows);
    if (sz_b < ld_b && Z > 1) {  // keep strides monotonic: dims (k, z, r)
        const uint64_t dims[3] = {uint64_t(K), uint64_t(Z), uint64_t(rows)};
        const uint64_t strides[2] = {sz_b, ld_b};
        const uint32_t box[3] = {uint32_t(kBK), 1, box_rows};
        *zr_order = 1;
        return make_tmap_bf16(base, 3, dims, strides, box);
    }
    const uint64_t dims[3] = {uint64_t(K), uint64_t(rows), uint64_t(Z)};
    const uint64_t strides[2] = {ld_b, sz_b};
    const uint32_t box[3] = {uint32_t(kBK), box_rows, 1};
    *zr_order = 0;
    return make_tmap_bf16(base, 3, dims, strides, box);
}

template <int BN>
void launch_bn(const GemmArgs& g, cudaStream_t st) {
    GemmParams p{};
    p.M = g.M, p.N = g.N, p.K = g.K, p.alpha = g.alpha, p.bias = g.bias, p.sbz = g.sbz;
    p.C = static_cast<__nv_bfloat16*>(g.C), p.ldc = g.ldc, p.sCz = g.sCz;
    CUtensorMap ta = operand_map(g.A, g.lda, g.sAz, g.M, g.K, g.Z, kBM, &p.a_zm);
    CUtensorMap tb = operand_map(g.B, g.ldb, g.sBz, g.N, g.K, g.Z, BN, &p.b_zm);
    auto kern = tc_gemm_kernel<BN>;
    constexpr uint32_t smem = GemmSmem<BN>::kTotal;
    ELA_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    dim3 grid(unsigned(ceil_div(g.N, BN)), unsigned(ceil_div(g.M, kBM)), unsigned(g.Z));
    kern<<<grid, 128, smem, st>>>(ta, tb, p);
    ELA_CHECK_LAUNCH();
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

bool tc_gemm_supported(const GemmArgs& g) {
    return g.K % kBK == 0 && g.K > 0 && g.N % 16 == 0 && g.M > 0 && g.lda % 8 == 0 && g.ldb % 8 == 0 &&
           g.ldc % 8 == 0 && g.sAz % 8 == 0 && g.sBz % 8 == 0 && g.sCz % 8 == 0 && aligned16(g.A) &&
           aligned16(g.B) && aligned16(g.C);
}

void launch_tc_gemm(const GemmArgs& g, cudaStream_t st) {
    if (g.N <= 64)
        launch_bn<64>(g, st);
    else
        launch_bn<128>(g, st);
}

}  // namespace elattn_gpu
