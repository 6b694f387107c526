// tf32_gemm.cu — the fp32 path's GEMMs on the tensor cores (tcgen05.mma kind::tf32) at
// fp32 accuracy ("3xTF32"):
//
//   C[z][m][n] = alpha * sum_k (A_hi B_hi + A_hi B_lo + A_lo B_hi)[z][m][n][k] + bias[z][n]
//
// where X_hi = tf32(X) (round to nearest) and X_lo = X - X_hi (exact in fp32; the tensor
// core reads its top 10 mantissa bits).  The dropped A_lo B_lo term and the truncation of
// the lo parts are ~2^-22 relative per product, so the fp32 path keeps the reference's
// 1e-5 gate (its f32 mode drifts 1.6e-7) at tensor-core rates instead of
// FFMA.  The three products are three K-SEGMENTS of one accumulation: segment s streams the
// (A_{hi|hi|lo}, B_{hi|lo|hi}) tensor-map pair, so no concatenated operand is ever
// materialised; producers of intermediates write hi/lo pairs directly (OUT_SPLIT epilogue),
// and tf32_split_kernel splits fp32 inputs.
//
// Used for the fp32 path of every stage (attention.hpp:197-290 at the reference's f32
// precision class): Q = Y.W_Q + b_Q, q'_i = Q_i.W_K,i^T, the decode as S = q'.H^T (B K-major)
// and C = P.H (B = H read MN-major), V_i = C_i.W_V,i + b_V,i, out = V.W_O + b_O.
//
// Structure as tc_gemm.cu (persistent, warp-specialised; warp 0 TMA, warp 1 MMA, warps 2..9
// epilogue), with fp32 operands: a k-block is 32 elements (one 128-byte SWIZZLE_128B row),
// one MMA covers K = 8, a stage carries one k-block of A_hi, A_lo, B_hi and B_lo.
#include "common.cuh"
#include "kernels.h"
#include "ptx_sm100.cuh"
#include "tmap.h"

namespace elattn_gpu {

namespace {

constexpr int kBM = 128, kBK = 32, kKBP = 1;
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;

__host__ __device__ constexpr uint32_t idesc_tf32(uint32_t M, uint32_t N, uint32_t a_mn, uint32_t b_mn) {
    // kind::tf32: c_format F32 (1), a/b format TF32 (2), majors, N >> 3, M >> 4
    return (1u << 4) | (2u << 7) | (2u << 10) | (a_mn << 15) | (b_mn << 16) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ float tf32_hi(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

template <int BN>
struct Tf32Smem {
    static constexpr uint32_t kABytes = kBM * kBK * 4;  // 16 KB: one k-block of A (hi or lo)
    static constexpr uint32_t kBBytes = BN * kBK * 4;   // one k-block of B (hi or lo)
    static constexpr uint32_t kStageBytes = 2 * kABytes + 2 * kBBytes;  // A_hi, A_lo, B_hi, B_lo
    static constexpr uint32_t kSliceBytes = 32 * 128;  // per epilogue warp: 32 rows x 32 fp32
    static constexpr uint32_t kOutBytes = kEpiWarps * kSliceBytes;
    static constexpr int kStagesFit = int((232448u - kOutBytes - 256 - 1024) / kStageBytes);
    static constexpr int kStages = kStagesFit < 6 ? kStagesFit : 6;
    static constexpr uint32_t kOutOff = kStages * kStageBytes;
    static constexpr uint32_t kBarOff = kOutOff + kOutBytes;
    static constexpr uint32_t kTotal = kBarOff + 256 + 1024;
    static constexpr uint32_t kTmemCols = 2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512);
    static_assert(kStages >= 2, "smem ring");
};

struct Tf32Params {
    int M, N, K, Z;
    int tiles_m, tiles_n;
    float alpha;
    const float* bias;
    int64_t sbz;
    int a_zm, b_zm;  // 1: map coordinate order (k, z, rows, kb) instead of (k, rows, z, kb)
    int a_bcast;
    int pdl;
    float* C;        // hi (or the only) output: C + z * sCz + m * ldc + n
    float* C_lo;     // SPLIT: the lo parts
    int64_t ldc, sCz;
};

// Operands are K-major (kind::tf32 with an MN-major SWIZZLE_128B B operand measured wrong
// on B200, so the decode's C = P.H reads a transposed hi/lo copy of H, tf32_split_t_kernel).
//
// Accuracy: the tensor core rounds its fp32 accumulator toward zero at every MMA, so a long
// chain of MMAs into one TMEM accumulator loses ~2^-24 relative per step, linearly in K
// (measured: 1e-5 at K = 1024 for one 3xTF32 chain, tools/tf32_diag.py).  Each 32-wide
// k-block is therefore its own short chain (12 MMAs: the three hi/lo products, K = 8 each)
// in a double-buffered TMEM chunk accumulator, and the epilogue warps sum the chunks in
// fp32 registers (round to nearest).
template <int BN, bool SPLIT, bool BIAS>
__global__ void __launch_bounds__(kThreads, 1)
    tf32x3_gemm_kernel(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmA1,
                       const __grid_constant__ CUtensorMap tmB0, const __grid_constant__ CUtensorMap tmB1,
                       Tf32Params p) {
    using S = Tf32Smem<BN>;
    constexpr int kStages = S::kStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* out_stage = smem + S::kOutOff;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kBarOff);
    uint64_t* empty = full + kStages;
    uint64_t* acc_full = empty + kStages;
    uint64_t* acc_empty = acc_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

    const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
    const int num_kb = p.K / kBK;
    const int num_tiles = p.Z * p.tiles_m * p.tiles_n;
    auto tile_coords = [&](int t, int& z, int& m0, int& n0) {
        z = t % p.Z;
        const int r = t / p.Z;
        m0 = (r / p.tiles_n) * kBM;
        n0 = (r % p.tiles_n) * BN;
    };

    if (warp == 0) {
        if (ptx::elect_one()) {
            ptx::prefetch_tmap(&tmA0);
            ptx::prefetch_tmap(&tmA1);
            ptx::prefetch_tmap(&tmB0);
            ptx::prefetch_tmap(&tmB1);
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
    if (p.pdl) {
        ptx::griddep_launch_dependents();
        ptx::griddep_wait();
    }

    if (warp == 0) {
        // ---- TMA producer: per k-block one stage {A_hi, A_lo, B_hi, B_lo}
        if (ptx::elect_one()) {
            int it = 0;
            for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
                int z, m0, n0;
                tile_coords(t, z, m0, n0);
                const int za = p.a_bcast ? 0 : z;
                for (int kb = 0; kb < num_kb; ++kb, ++it) {
                    const int s = it % kStages;
                    ptx::mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
                    uint8_t* a = smem + s * S::kStageBytes;
                    uint8_t* b = a + 2 * S::kABytes;
                    ptx::mbar_arrive_expect_tx(&full[s], S::kStageBytes);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const CUtensorMap* ta = h ? &tmA1 : &tmA0;
                        const CUtensorMap* tb = h ? &tmB1 : &tmB0;
                        if (p.a_zm)
                            ptx::tma_load_4d(a + h * S::kABytes, ta, &full[s], 0, za, m0, kb, ptx::kEvictNormal);
                        else
                            ptx::tma_load_4d(a + h * S::kABytes, ta, &full[s], 0, m0, za, kb, ptx::kEvictNormal);
                        if (p.b_zm) {
                            ptx::tma_load_4d(b + h * S::kBBytes, tb, &full[s], 0, z, n0, kb, ptx::kEvictNormal);
                        } else {
                            ptx::tma_load_4d(b + h * S::kBBytes, tb, &full[s], 0, n0, z, kb, ptx::kEvictNormal);
                        }
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ---- MMA issuer: one chunk (12 MMAs: A_hi B_hi, A_hi B_lo, A_lo B_hi; K = 8 each) per
        // k-block into TMEM chunk buffer (chunk & 1)
        constexpr uint32_t idesc = idesc_tf32(kBM, BN, 0, 0);
        const uint32_t sbase = ptx::smem_u32(smem);
        int it = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
            for (int kb = 0; kb < num_kb; ++kb, ++it) {
                const int ab = it & 1;
                ptx::mbar_wait(&acc_empty[ab], ((it >> 1) & 1) ^ 1);
                const int s = it % kStages;
                ptx::mbar_wait(&full[s], (it / kStages) & 1);
                ptx::tc_fence_after();
                if (lane == 0) {
                    const uint32_t a_addr = sbase + s * S::kStageBytes;
                    const uint32_t b_addr = a_addr + 2 * S::kABytes;
#pragma unroll
                    for (int sg = 0; sg < 3; ++sg) {
                        const uint32_t aa = a_addr + (sg == 2 ? S::kABytes : 0);
                        const uint32_t ba = b_addr + (sg == 1 ? S::kBBytes : 0);
#pragma unroll
                        for (int k = 0; k < kBK / 8; ++k) {  // K = 8 per MMA = 32 bytes along K
                            const uint64_t ad = ptx::sdesc_sw128(aa + 32 * k, 0, 1024);
                            const uint64_t bd = ptx::sdesc_sw128(ba + 32 * k, 0, 1024);
                            mma_tf32(tmem + ab * BN, ad, bd, idesc, (sg | k) != 0);
                        }
                    }
                    ptx::mma_commit(&empty[s]);
                    ptx::mma_commit(&acc_full[ab]);
                }
                __syncwarp();
            }
        }
    } else {
        // ---- epilogue: warp (qd = warp % 4, column half g) owns 32 rows x BN/2 columns;
        // it sums the k-block chunks in registers, then adds bias, writes through its smem
        // slice with coalesced st.global.v4 (4 rows x 128 B per instruction); SPLIT writes
        // hi and lo parts
        const uint32_t qd = warp & 3, grp = (warp - 2) >> 2;
        constexpr int kHalf = BN / 2;
        uint8_t* slice = out_stage + (warp - 2) * S::kSliceBytes;
        int it = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
            int z, m0, n0;
            tile_coords(t, z, m0, n0);
            float acc[kHalf];
#pragma unroll
            for (int j = 0; j < kHalf; ++j) acc[j] = 0.f;
            for (int kb = 0; kb < num_kb; ++kb, ++it) {
                const int ab = it & 1;
                ptx::mbar_wait(&acc_full[ab], (it >> 1) & 1);
                ptx::tc_fence_after();
                uint32_t rr[kHalf];
#pragma unroll
                for (int c0 = 0; c0 < kHalf; c0 += 32)
                    ptx::tmem_ld32(tmem + ((qd * 32) << 16) + ab * BN + grp * kHalf + c0,
                                   *reinterpret_cast<uint32_t(*)[32]>(&rr[c0]));
                ptx::tmem_ld_wait();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&acc_empty[ab]);
#pragma unroll
                for (int j = 0; j < kHalf; ++j) acc[j] += __uint_as_float(rr[j]);
            }
            const int rbase = m0 + int(qd) * 32;
#pragma unroll
            for (int c0 = 0; c0 < kHalf; c0 += 32) {
                const int nb = n0 + int(grp) * kHalf + c0;
                float v[32];
                const float bc = BIAS ? ((nb + int(lane) < p.N) ? __ldg(p.bias + z * p.sbz + nb + lane) : 0.f) : 0.f;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    v[j] = acc[c0 + j] * p.alpha;
                    if constexpr (BIAS) v[j] += __shfl_sync(0xffffffffu, bc, j);
                }
#pragma unroll
                for (int part = 0; part < (SPLIT ? 2 : 1); ++part) {
                    float* dst = part == 0 ? p.C : p.C_lo;
                    // row = lane: 8 chunks of 16 bytes, chunk c at c ^ (lane & 7)
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        float4 w;
                        float* wf = reinterpret_cast<float*>(&w);
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const float x = v[4 * q + u];
                            if constexpr (SPLIT) {
                                const float hi = tf32_hi(x);
                                wf[u] = part == 0 ? hi : x - hi;
                            } else {
                                wf[u] = x;
                            }
                        }
                        *reinterpret_cast<float4*>(slice + lane * 128 + ((q ^ (lane & 7)) << 4)) = w;
                    }
                    __syncwarp();
#pragma unroll
                    for (int s4 = 0; s4 < 8; ++s4) {
                        const int r = s4 * 4 + int(lane >> 3), ch = int(lane & 7);
                        const float4 w = *reinterpret_cast<const float4*>(slice + r * 128 + ((ch ^ (r & 7)) << 4));
                        const int row = rbase + r, col = nb + 4 * ch;
                        if (row < p.M && col < p.N)
                            *reinterpret_cast<float4*>(dst + z * p.sCz + int64_t(row) * p.ldc + col) = w;
                    }
                    __syncwarp();
                }
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<S::kTmemCols>(tmem);
    }
}

// fp32 tensor maps (32-element = 128-byte k-blocks, SWIZZLE_128B)
CUtensorMap f32_map(const void* base, int rank, const uint64_t* dims, const uint64_t* strides, const uint32_t* box) {
    return make_tmap(base, 4, rank, dims, strides, box, 128);
}

// K-major operand X[z][r][k]: 4-D (32 k, r | z, z | r, k-block), box (32, box_rows, 1, KBP)
CUtensorMap kmajor_map(const float* base, int64_t ld, int64_t sz, int rows, int K, int Z, uint32_t box_rows,
                       int* zr_order) {
    uint64_t ld_b = uint64_t(ld) * 4, sz_b = uint64_t(sz) * 4;
    if (Z == 1 || sz == 0) sz_b = ld_b * uint64_t(rows);
    *zr_order = (sz_b < ld_b && Z > 1) ? 1 : 0;
    const uint64_t nkb = uint64_t((K + kBK - 1) / kBK);
    if (*zr_order) {
        const uint64_t dims[4] = {uint64_t(kBK), uint64_t(Z), uint64_t(rows), nkb};
        const uint64_t strides[3] = {sz_b, ld_b, uint64_t(kBK) * 4};
        const uint32_t box[4] = {uint32_t(kBK), 1, box_rows, uint32_t(kKBP)};
        return f32_map(base, 4, dims, strides, box);
    }
    const uint64_t dims[4] = {uint64_t(kBK), uint64_t(rows), uint64_t(Z), nkb};
    const uint64_t strides[3] = {ld_b, sz_b, uint64_t(kBK) * 4};
    const uint32_t box[4] = {uint32_t(kBK), box_rows, 1, uint32_t(kKBP)};
    return f32_map(base, 4, dims, strides, box);
}

int num_sms_tf32() {
    static int n = [] {
        int dev = 0, v = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return n;
}

template <int BN, bool SPLIT, bool BIAS>
void launch_t(const Tf32GemmArgs& g, cudaStream_t st) {
    using S = Tf32Smem<BN>;
    Tf32Params p{};
    p.M = g.M, p.N = g.N, p.K = g.K, p.Z = g.Z, p.alpha = g.alpha, p.bias = g.bias, p.sbz = g.sbz;
    p.tiles_m = int(ceil_div(g.M, kBM));
    p.tiles_n = int(ceil_div(g.N, BN));
    p.a_bcast = (g.Z > 1 && g.sAz == 0) ? 1 : 0;
    p.pdl = pdl_enabled() ? 1 : 0;
    p.C = g.C, p.C_lo = g.C_lo, p.ldc = g.ldc, p.sCz = g.sCz;
    const int Za = p.a_bcast ? 1 : g.Z;
    int zr = 0;
    CUtensorMap ta0 = kmajor_map(g.A_hi, g.lda, g.sAz, g.M, g.K, Za, kBM, &p.a_zm);
    CUtensorMap ta1 = kmajor_map(g.A_lo, g.lda, g.sAz, g.M, g.K, Za, kBM, &zr);
    CUtensorMap tb0 = kmajor_map(g.B_hi, g.ldb, g.sBz, g.N, g.K, g.Z, BN, &p.b_zm);
    CUtensorMap tb1 = kmajor_map(g.B_lo, g.ldb, g.sBz, g.N, g.K, g.Z, BN, &zr);
    auto kern = tf32x3_gemm_kernel<BN, SPLIT, BIAS>;
    ELA_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(S::kTotal)));
    const int tiles = p.Z * p.tiles_m * p.tiles_n;
    const int grid = tiles < num_sms_tf32() ? tiles : num_sms_tf32();
    launch_ex(kern, dim3(grid), dim3(kThreads), S::kTotal, st, 1, ta0, ta1, tb0, tb1, p);
    ELA_CHECK_LAUNCH();
}

template <int BN>
void launch_bn(const Tf32GemmArgs& g, cudaStream_t st) {
    const bool split = g.C_lo != nullptr, bias = g.bias != nullptr;
    if (split) return bias ? launch_t<BN, true, true>(g, st) : launch_t<BN, true, false>(g, st);
    return bias ? launch_t<BN, false, true>(g, st) : launch_t<BN, false, false>(g, st);
}

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

bool tf32_gemm_supported(const Tf32GemmArgs& g) {
    const bool base = g.M > 0 && g.N > 0 && g.K > 0 && g.K % kBK == 0 && g.N % 4 == 0 && g.lda % 4 == 0 &&
                      g.ldb % 4 == 0 && g.ldc % 4 == 0 && g.sAz % 4 == 0 && g.sBz % 4 == 0 && g.sCz % 4 == 0 &&
                      al16(g.A_hi) && al16(g.A_lo) && al16(g.B_hi) && al16(g.B_lo) && al16(g.C) &&
                      (g.C_lo == nullptr || al16(g.C_lo));
    return base;
}

void launch_tf32_gemm(const Tf32GemmArgs& g, cudaStream_t st) {
    ELA_REQUIRE(tf32_gemm_supported(g), ELATTN_ERR_UNSUPPORTED, "tf32 GEMM: shape outside the envelope");
    if (g.N <= 64)
        launch_bn<64>(g, st);
    else
        launch_bn<128>(g, st);
}

// X -> (tf32(X), X - tf32(X)) for `rows` rows of `cols` fp32 (row stride ld); rows r with
// (npi and r % n_stride >= npi[r / n_stride]) are zeroed (ragged padding of H).
__global__ void tf32_split_kernel(const float* __restrict__ X, int64_t rows, int cols, int64_t ld,
                                  float* __restrict__ hi, float* __restrict__ lo, const int* __restrict__ npi,
                                  int n_stride, const int* __restrict__ h_index) {
    const int64_t total4 = rows * (cols / 4);
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total4; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = e / (cols / 4);
        const int c = int(e % (cols / 4)) * 4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        const bool keep = npi == nullptr || int(r % n_stride) < npi[r / n_stride];
        // slot-indexed H: block b of the output reads block h_index[b] of X
        const int64_t rs = h_index ? int64_t(h_index[r / n_stride]) * n_stride + r % n_stride : r;
        if (keep) v = *reinterpret_cast<const float4*>(X + rs * ld + c);
        float4 h, l;
        h.x = tf32_hi(v.x), h.y = tf32_hi(v.y), h.z = tf32_hi(v.z), h.w = tf32_hi(v.w);
        l.x = v.x - h.x, l.y = v.y - h.y, l.z = v.z - h.z, l.w = v.w - h.w;
        *reinterpret_cast<float4*>(hi + r * cols + c) = h;
        *reinterpret_cast<float4*>(lo + r * cols + c) = l;
    }
}

// H [B][n][d_m] -> (tf32(H^T), H^T - tf32(H^T)) [B][d_m][n_pad]: the K-major B operand of
// C = P.H (keys = K).  Keys t >= n_b (ragged) or t >= n (padding up to n_pad) are zero.
__global__ void tf32_split_t_kernel(const float* __restrict__ H, int n, int d_m, int n_pad,
                                    const int* __restrict__ npi, float* __restrict__ hi, float* __restrict__ lo,
                                    const int* __restrict__ h_index) {
    __shared__ float tile[32][33];
    const int b = blockIdx.z, t0 = blockIdx.x * 32, d0 = blockIdx.y * 32;
    const int n_b = npi ? npi[b] : n;
    const float* Hb = H + int64_t(h_index ? h_index[b] : b) * n * d_m;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int t = t0 + r, d = d0 + threadIdx.x;
        tile[r][threadIdx.x] = (t < n && t < n_b && d < d_m) ? Hb[int64_t(t) * d_m + d] : 0.f;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int d = d0 + r, t = t0 + threadIdx.x;
        if (d < d_m && t < n_pad) {
            const float v = tile[threadIdx.x][r];
            const float h = tf32_hi(v);
            const int64_t o = (int64_t(b) * d_m + d) * n_pad + t;
            hi[o] = h;
            lo[o] = v - h;
        }
    }
}

void launch_tf32_split_t(const float* H, int B, int n, int d_m, int n_pad, const int* npi, float* hi, float* lo,
                         cudaStream_t st, const int* h_index) {
    dim3 grid(unsigned((n_pad + 31) / 32), unsigned((d_m + 31) / 32), unsigned(B));
    tf32_split_t_kernel<<<grid, dim3(32, 8), 0, st>>>(H, n, d_m, n_pad, npi, hi, lo, h_index);
    ELA_CHECK_LAUNCH();
}

void launch_tf32_split(const float* X, int64_t rows, int cols, int64_t ld, float* hi, float* lo, const int* npi,
                       int n_stride, cudaStream_t st, const int* h_index) {
    ELA_REQUIRE(cols % 4 == 0 && ld % 4 == 0, ELATTN_ERR_UNSUPPORTED, "tf32 split: cols must be a multiple of 4");
    const int64_t total4 = rows * (cols / 4);
    const int grid = int(std::min<int64_t>((total4 + 255) / 256, int64_t(num_sms_tf32()) * 8));
    tf32_split_kernel<<<grid > 0 ? grid : 1, 256, 0, st>>>(X, rows, cols, ld, hi, lo, npi, n_stride, h_index);
    ELA_CHECK_LAUNCH();
}

// Softmax of score rows S [B][rows][ld] (raw q'.H^T) over the first n_b keys of input b,
// scale folded into exp2: P = 2^(s * c - m) / l with c = scale * log2(e), written as
// (P_hi, P_lo) [B][rows][ld] with zeros for keys >= n_b; stats (optional) {m, l} per row
// in log2 units (as the bf16 decode's).  One warp per row.
__global__ void tf32_softmax_kernel(const float* __restrict__ S, int64_t total_rows, int rows, int n_stride, int ld,
                                    const int* __restrict__ npi, float scale_log2, float* __restrict__ P_hi,
                                    float* __restrict__ P_lo, float2* __restrict__ stats) {
    const int64_t row = blockIdx.x * int64_t(blockDim.x / 32) + threadIdx.x / 32;
    if (row >= total_rows) return;
    const int lane = threadIdx.x % 32;
    const int b = int(row / rows);
    const int n_b = npi ? npi[b] : n_stride;
    const float* s = S + row * ld;
    float m = -INFINITY;
    for (int j = lane; j < n_b; j += 32) m = fmaxf(m, s[j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    const float ms = m * scale_log2;
    float l = 0.f;
    for (int j = lane; j < n_b; j += 32) l += exp2f(fmaf(s[j], scale_log2, -ms));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    const bool bad = n_b < 1 || n_b > n_stride;  // out-of-contract length: loud NaN rows
    const float inv = bad ? __int_as_float(0x7fc00000) : 1.f / l;
    for (int j = lane; j < ld; j += 32) {
        const float pv = j < n_b ? exp2f(fmaf(s[j], scale_log2, -ms)) * inv : (bad ? inv : 0.f);
        const float hi = tf32_hi(pv);
        P_hi[row * ld + j] = hi;
        P_lo[row * ld + j] = pv - hi;
    }
    if (stats != nullptr && lane == 0) stats[row] = make_float2(ms, l);
}

void launch_tf32_softmax(const float* S, int64_t total_rows, int rows, int n_stride, int ld, const int* npi,
                         float scale, float* P_hi, float* P_lo, float2* stats, cudaStream_t st) {
    const int warps = 8;
    const int64_t grid = (total_rows + warps - 1) / warps;
    tf32_softmax_kernel<<<unsigned(grid), 32 * warps, 0, st>>>(S, total_rows, rows, n_stride, ld, npi,
                                                               scale * 1.4426950408889634f, P_hi, P_lo, stats);
    ELA_CHECK_LAUNCH();
}

}  // namespace elattn_gpu
