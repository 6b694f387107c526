// el_decode_tc.cu — the fused EL-attention decode kernel for sm_100a (bf16).
//
// Computes, for every input b and each of its `rows` (= beams x heads) EL-Q rows,
//     C = softmax(q' . H_b^T / sqrt(d_k)) . H_b                      (fp32 accumulate)
// i.e. the core of el_attention_folded (attention.hpp:272-280), reading H_b from
// HBM exactly once and using every staged tile as BOTH key and value.
//
// Work split — one thread-block CLUSTER of 2 CTAs per input, split along d_m:
//   CTA r owns d_m columns [r*d_m/2, (r+1)*d_m/2).  Its EL-Q half q'_r (64 x d_m/2)
//   stays resident in smem; H_b streams through a TMA ring in tiles of 32 rows x
//   d_m/2 (SWIZZLE_128B, 128-column "units" of 8 KB).
//   Per tile j:
//     S_r   = q'_r . H_tile,r^T         tcgen05.mma M=64 N=32, K = d_m/2   (TMEM)
//     S     = S_0 + S_1                  partial scores swapped through DSMEM
//                                        (st.async + mbarrier complete_tx)
//     P     = exp2(S*scale*log2e - m)    online softmax, one query row per thread,
//                                        lazy rescale (FA4-style threshold 2^8)
//     O_r^T += H_tile,r^T . P^T          tcgen05.mma M=128 (d_m) N=64 (queries),
//                                        A = the SAME smem tile read MN-major
//   O_r (d_m/2 x 64 fp32) lives in TMEM for the whole input; the epilogue divides
//   by the softmax sums and writes C rows b*rows + q, columns of this CTA's half.
// Both CTAs see bit-identical S (fp32 add commutes), so their softmax decisions agree.
//
// Roles (192 threads): warp 0 TMA producer, warp 1 MMA issuer (+TMEM owner),
// warps 2..5 softmax / rescale / epilogue (TMEM lane quadrant = warp % 4).
#include "common.cuh"
#include "kernels.h"
#include "ptx_sm100.cuh"
#include "tmap.h"

namespace elattn_gpu {

namespace {

constexpr int kRowsQ = 64;     // EL-Q rows per input (padded)
constexpr int kNT = 32;        // H rows per tile
constexpr int kRing = 12;      // 8 KB units in the H ring
constexpr int kUnitBytes = 8192;   // 32 rows x 128 d_m x bf16
constexpr int kChunkBytes = 4096;  // 32 rows x 64 d_m
constexpr int kThreads = 192;
constexpr float kRescaleThreshold = 8.0f;  // log2 domain: rescale only when max grows by > 2^8

template <int UNITS>  // 128-column units per CTA: d_m = 256 * UNITS
struct DecSmem {
    static constexpr uint32_t kQBytes = UNITS * 2 * 8192;        // 64 rows x d_m/2
    static constexpr uint32_t kRingOff = kQBytes;
    static constexpr uint32_t kPOff = kRingOff + kRing * kUnitBytes;  // 2 x (64 rows x 128 B)
    static constexpr uint32_t kRecvOff = kPOff + 2 * 8192;            // 2 x (64 x 32 fp32)
    static constexpr uint32_t kAlphaOff = kRecvOff + 2 * 8192;        // 2 x 64 fp32
    static constexpr uint32_t kLOff = kAlphaOff + 2 * 64 * 4;         // 64 fp32
    static constexpr uint32_t kBarOff = kLOff + 64 * 4;
    static constexpr int kNumBars = 1 + 2 * kRing + 2 * 5 + 2;
    static constexpr uint32_t kTotal = kBarOff + kNumBars * 8 + 16 + 1024;
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

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
}

template <int UNITS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    el_decode_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_h,
                        const int* __restrict__ n_per_input, int rows, int n_stride, int d_m, float scale_log2,
                        __nv_bfloat16* __restrict__ ctx) {
    using L = DecSmem<UNITS>;
    constexpr int kTmemCols = 512;
    constexpr uint32_t kTmemS = 256;  // S double buffer at columns 256..319
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sq = smem;
    uint8_t* ring = smem + L::kRingOff;
    uint8_t* sP = smem + L::kPOff;
    float* recv = reinterpret_cast<float*>(smem + L::kRecvOff);
    float* s_alpha = reinterpret_cast<float*>(smem + L::kAlphaOff);
    float* s_l = reinterpret_cast<float*>(smem + L::kLOff);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
    uint64_t* q_full = bars;
    uint64_t* unit_full = bars + 1;
    uint64_t* unit_empty = unit_full + kRing;
    uint64_t* s_full = unit_empty + kRing;
    uint64_t* s_empty = s_full + 2;
    uint64_t* p_full = s_empty + 2;
    uint64_t* p_empty = p_full + 2;
    uint64_t* recv_full = p_empty + 2;
    uint64_t* o_done = recv_full + 2;
    uint64_t* o_full = o_done + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 1);

    const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
    const uint32_t rank = ptx::cluster_ctarank(), peer = rank ^ 1u;
    const int b = blockIdx.x >> 1;
    const int dm_half = d_m / 2, dm_off = int(rank) * dm_half;
    const int n_b = n_per_input ? n_per_input[b] : n_stride;
    const bool valid = n_b >= 1 && n_b <= n_stride;
    const int T = valid ? (n_b + kNT - 1) / kNT : 0;

    if (warp == 0) {
        if (ptx::elect_one()) {
            ptx::prefetch_tmap(&tm_q);
            ptx::prefetch_tmap(&tm_h);
            ptx::mbar_init(q_full, 1);
            for (int s = 0; s < kRing; ++s) {
                ptx::mbar_init(&unit_full[s], 1);
                ptx::mbar_init(&unit_empty[s], 1);
            }
            for (int i = 0; i < 2; ++i) {
                ptx::mbar_init(&s_full[i], 1);
                ptx::mbar_init(&s_empty[i], 4);
                ptx::mbar_init(&p_full[i], 4);
                ptx::mbar_init(&p_empty[i], 1);
                ptx::mbar_init(&recv_full[i], 1);
            }
            ptx::mbar_init(o_done, 1);
            ptx::mbar_init(o_full, 1);
            ptx::fence_mbar_init();
        }
        __syncwarp();
    } else if (warp == 1) {
        ptx::tmem_alloc<kTmemCols>(tmem_slot);
    }
    ptx::tc_fence_before();
    ptx::cluster_sync();  // peer barriers initialised before any st.async targets them
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ================= TMA producer =================
        if (ptx::elect_one() && T > 0) {
            ptx::mbar_arrive_expect_tx(q_full, L::kQBytes);
            for (int c = 0; c < 2 * UNITS; ++c)
                ptx::tma_load_2d(sq + c * 8192, &tm_q, q_full, dm_off + 64 * c, b * rows, ptx::kEvictNormal);
            for (int j = 0; j < T; ++j) {
                for (int u = 0; u < UNITS; ++u) {
                    const int g = j * UNITS + u, s = g % kRing;
                    ptx::mbar_wait(&unit_empty[s], ((g / kRing) & 1) ^ 1);
                    uint8_t* dst = ring + s * kUnitBytes;
                    ptx::mbar_arrive_expect_tx(&unit_full[s], kUnitBytes);
                    const int col = dm_off + 128 * u;
                    ptx::tma_load_3d(dst, &tm_h, &unit_full[s], col, j * kNT, b, ptx::kEvictFirst);
                    ptx::tma_load_3d(dst + kChunkBytes, &tm_h, &unit_full[s], col + 64, j * kNT, b,
                                     ptx::kEvictFirst);
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ================= MMA issuer =================
        if (ptx::elect_one() && T > 0) {
            constexpr uint32_t idS = ptx::idesc_bf16(64, kNT, 0, 0);    // S = q' . H^T
            constexpr uint32_t idO = ptx::idesc_bf16(128, 64, 1, 0);    // O^T += H^T . P^T (A MN-major)
            const uint32_t q_base = ptx::smem_u32(sq), ring_base = ptx::smem_u32(ring), p_base = ptx::smem_u32(sP);
            auto issue_O = [&](int t) {
                const int pb = t & 1;
                ptx::mbar_wait(&p_full[pb], (t >> 1) & 1);
                ptx::tc_fence_after();
#pragma unroll
                for (int m = 0; m < UNITS; ++m) {
                    const int s = (t * UNITS + m) % kRing;
#pragma unroll
                    for (int kk = 0; kk < kNT / 16; ++kk) {
                        const uint64_t a = ptx::sdesc_sw128(ring_base + s * kUnitBytes + kk * 2048, kChunkBytes, 1024);
                        const uint64_t bd = ptx::sdesc_sw128(p_base + pb * 8192 + 32 * kk, 0, 1024);
                        ptx::mma_bf16(tmem + m * 64, a, bd, idO, (t > 0 || kk > 0) ? 1u : 0u);
                    }
                    ptx::mma_commit(&unit_empty[s]);
                }
                ptx::mma_commit(&p_empty[pb]);
                ptx::mma_commit(o_done);
            };
            ptx::mbar_wait(q_full, 0);
            for (int j = 0; j < T; ++j) {
                const int sb = j & 1;
                ptx::mbar_wait(&s_empty[sb], ((j >> 1) & 1) ^ 1);
                ptx::tc_fence_after();
#pragma unroll
                for (int u = 0; u < UNITS; ++u) {
                    const int g = j * UNITS + u, s = g % kRing;
                    ptx::mbar_wait(&unit_full[s], (g / kRing) & 1);
                    ptx::tc_fence_after();
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const int h = kk >> 2, k16 = kk & 3;
                        const uint64_t a = ptx::sdesc_sw128(q_base + (2 * u + h) * 8192 + 32 * k16, 0, 1024);
                        const uint64_t bd =
                            ptx::sdesc_sw128(ring_base + s * kUnitBytes + h * kChunkBytes + 32 * k16, 0, 1024);
                        ptx::mma_bf16(tmem + kTmemS + sb * kNT, a, bd, idS, (u | kk) != 0 ? 1u : 0u);
                    }
                }
                ptx::mma_commit(&s_full[sb]);
                if (j >= 1) issue_O(j - 1);
            }
            issue_O(T - 1);
            ptx::mma_commit(o_full);
        }
        __syncwarp();
    } else {
        // ================= softmax / rescale / epilogue (warps 2..5) =================
        const uint32_t qd = warp & 3;          // TMEM lane quadrant of this warp
        const int q = int(qd) * 16 + int(lane);  // query row owned (lanes 0..15, M=64 layout)
        const bool owner = lane < 16;
        const uint32_t t_lane = tmem + ((qd * 32) << 16);
        const uint32_t recv_base = ptx::smem_u32(recv);
        float m_used = -INFINITY, l_sum = 0.f;
        const bool zero_tail = (n_per_input != nullptr) && (T * kNT > n_b);
        for (int j = 0; j < T; ++j) {
            const int sb = j & 1;
            const uint32_t par = (j >> 1) & 1;
            if (warp == 2 && lane == 0) ptx::mbar_arrive_expect_tx(&recv_full[sb], kRowsQ * kNT * 4);
            ptx::mbar_wait(&s_full[sb], par);
            ptx::tc_fence_after();
            uint32_t sr[32];
            {
                uint32_t lo[16], hi[16];
                ptx::tmem_ld16(t_lane + kTmemS + sb * kNT, lo);
                ptx::tmem_ld16(t_lane + kTmemS + sb * kNT + 16, hi);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 16; ++i) sr[i] = lo[i], sr[16 + i] = hi[i];
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&s_empty[sb]);
            // swap partial scores with the peer CTA
            if (owner) {
                const uint32_t dst = ptx::mapa(recv_base + uint32_t((sb * kRowsQ + q) * kNT * 4), peer);
                const uint32_t rbar = ptx::mapa(ptx::smem_u32(&recv_full[sb]), peer);
#pragma unroll
                for (int i = 0; i < kNT; i += 4)
                    ptx::st_async_v4(dst + i * 4, __uint_as_float(sr[i]), __uint_as_float(sr[i + 1]),
                                     __uint_as_float(sr[i + 2]), __uint_as_float(sr[i + 3]), rbar);
            }
            ptx::mbar_wait(&recv_full[sb], par);
            uint32_t need = 0;
            uint32_t pk[16];
            if (owner) {
                const float4* pr = reinterpret_cast<const float4*>(recv + (sb * kRowsQ + q) * kNT);
                const int nvalid = min(kNT, n_b - j * kNT);
                float s[kNT];
#pragma unroll
                for (int i = 0; i < kNT / 4; ++i) {
                    const float4 v = pr[i];
                    s[4 * i + 0] = (__uint_as_float(sr[4 * i + 0]) + v.x) * scale_log2;
                    s[4 * i + 1] = (__uint_as_float(sr[4 * i + 1]) + v.y) * scale_log2;
                    s[4 * i + 2] = (__uint_as_float(sr[4 * i + 2]) + v.z) * scale_log2;
                    s[4 * i + 3] = (__uint_as_float(sr[4 * i + 3]) + v.w) * scale_log2;
                }
                float mt = -INFINITY;
#pragma unroll
                for (int i = 0; i < kNT; ++i) {
                    if (i >= nvalid) s[i] = -INFINITY;
                    mt = fmaxf(mt, s[i]);
                }
                float alpha = 1.f;
                if (mt > m_used + kRescaleThreshold) {
                    need = 1;
                    alpha = exp2f(m_used - mt);  // 0 on the first tile
                    l_sum *= alpha;
                    m_used = mt;
                }
                s_alpha[sb * 64 + q] = alpha;
                float acc = 0.f;
#pragma unroll
                for (int i = 0; i < kNT; i += 2) {
                    const float p0 = exp2f(s[i] - m_used), p1 = exp2f(s[i + 1] - m_used);
                    acc += p0 + p1;
                    pk[i / 2] = pack_bf16x2(p0, p1);
                }
                l_sum += acc;
            }
            // P[sb] is free once O(j-2) has consumed it
            ptx::mbar_wait(&p_empty[sb], par ^ 1);
            if (owner) {
                uint8_t* prow = sP + sb * 8192 + q * 128;
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    *reinterpret_cast<uint4*>(prow + ((c ^ (q & 7)) << 4)) =
                        make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
            }
            if (zero_tail && j == T - 1) {
                // rows n_b.. of the last tile are in-bounds padding of H_b: zero them
                // before they meet P = 0 in the MMA (0 * NaN would poison O).
                const int r0 = n_b - j * kNT;
                const int tid = int(threadIdx.x) - 64;
                for (int idx = tid; idx < UNITS * 2 * (kNT - r0) * 8; idx += 128) {
                    const int per_chunk = (kNT - r0) * 8;
                    const int ch = idx / per_chunk, rem = idx % per_chunk;
                    const int r = r0 + rem / 8, c16 = rem % 8;
                    const int s = (j * UNITS + ch / 2) % kRing;
                    *reinterpret_cast<uint4*>(ring + s * kUnitBytes + (ch & 1) * kChunkBytes + r * 128 + c16 * 16) =
                        make_uint4(0, 0, 0, 0);
                }
            }
            const uint32_t any = softmax_bar_or(need);
            if (any && j > 0) {
                // lazy rescale of the running O^T columns: wait for O(j-1), then O *= alpha
                ptx::mbar_wait(o_done, (j - 1) & 1);
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
        }
        // ---- epilogue: C[b*rows + q][dm_off + d] = O^T[d][q] / l_q
        if (owner) s_l[q] = l_sum;
        softmax_bar_sync();
        if (T > 0) {
            ptx::mbar_wait(o_full, 0);
            ptx::tc_fence_after();
        }
        const int d_local = int(qd) * 32 + int(lane);
        for (int m = 0; m < UNITS; ++m) {
            const int d = dm_off + m * 128 + d_local;
#pragma unroll
            for (int c0 = 0; c0 < 64; c0 += 16) {
                uint32_t r[16];
                if (T > 0) {
                    ptx::tmem_ld16(t_lane + m * 64 + c0, r);
                    ptx::tmem_ld_wait();
                }
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int qq = c0 + i;
                    if (qq < rows) {
                        const float v = T > 0 ? __uint_as_float(r[i]) / s_l[qq] : __int_as_float(0x7fc00000);
                        ctx[(int64_t(b) * rows + qq) * d_m + d] = __float2bfloat16_rn(v);
                    }
                }
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::cluster_sync();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<kTmemCols>(tmem);
    }
}

template <int UNITS>
void launch_units(const void* qp, const void* H, const int* npi, int B, int rows, int n_stride, int d_m,
                  float scale_log2, void* ctx, cudaStream_t st) {
    // q' viewed as [B*rows][d_m]; box 64 rows (rows < 64 pad with the next input's
    // rows or OOB zeros; only the first `rows` outputs are written).
    const uint64_t qdims[2] = {uint64_t(d_m), uint64_t(B) * rows};
    const uint64_t qstr[1] = {uint64_t(d_m) * 2};
    const uint32_t qbox[2] = {64, kRowsQ};
    CUtensorMap tq = make_tmap_bf16(qp, 2, qdims, qstr, qbox);
    const uint64_t hdims[3] = {uint64_t(d_m), uint64_t(n_stride), uint64_t(B)};
    const uint64_t hstr[2] = {uint64_t(d_m) * 2, uint64_t(n_stride) * d_m * 2};
    const uint32_t hbox[3] = {64, kNT, 1};
    CUtensorMap th = make_tmap_bf16(H, 3, hdims, hstr, hbox);
    auto kern = el_decode_tc_kernel<UNITS>;
    constexpr uint32_t smem = DecSmem<UNITS>::kTotal;
    ELA_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    kern<<<dim3(2 * B), kThreads, smem, st>>>(tq, th, npi, rows, n_stride, d_m, scale_log2,
                                               static_cast<__nv_bfloat16*>(ctx));
    ELA_CHECK_LAUNCH();
}

}  // namespace

bool el_decode_tc_supported(int rows_per_input, int d_m) {
    return rows_per_input >= 1 && rows_per_input <= kRowsQ && d_m % 256 == 0 && d_m >= 256 && d_m <= 1024;
}

void launch_el_decode_tc(const void* qp, const void* H, const int* n_per_input, int B, int rows_per_input,
                         int n_stride, int d_m, float scale, void* ctx, cudaStream_t st) {
    ELA_REQUIRE(el_decode_tc_supported(rows_per_input, d_m), ELATTN_ERR_UNSUPPORTED,
                "tcgen05 decode: rows <= 64 and d_m in {256, 512, 768, 1024}");
    ELA_REQUIRE((reinterpret_cast<uintptr_t>(qp) & 15) == 0 && (reinterpret_cast<uintptr_t>(H) & 15) == 0,
                ELATTN_ERR_PARAM, "tcgen05 decode: q' and H must be 16-byte aligned");
    const float scale_log2 = scale * 1.4426950408889634f;
    switch (d_m / 256) {
        case 1: return launch_units<1>(qp, H, n_per_input, B, rows_per_input, n_stride, d_m, scale_log2, ctx, st);
        case 2: return launch_units<2>(qp, H, n_per_input, B, rows_per_input, n_stride, d_m, scale_log2, ctx, st);
        case 3: return launch_units<3>(qp, H, n_per_input, B, rows_per_input, n_stride, d_m, scale_log2, ctx, st);
        default: return launch_units<4>(qp, H, n_per_input, B, rows_per_input, n_stride, d_m, scale_log2, ctx, st);
    }
}

}  // namespace elattn_gpu
