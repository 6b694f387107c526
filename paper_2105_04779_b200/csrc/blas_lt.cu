// blas_lt.cu — the two PLAIN projection GEMMs of a layer step (Q = Y.W_Q + b_Q and
// out = V.W_O + b_O, attention.hpp:205 / :283-288 with el_bias_terms :221-231) and the
// per-head V projection (strided batch over heads, :286) through cuBLASLt with a fused
// bias epilogue.  These are ordinary dense GEMMs (M = B*x rows,
// N = K = 1024 at BART shapes, 0.5 waves of 128x128 tiles on 148 SMs) where the library
// is faster than our persistent kernel; the EL-specific GEMMs (head-strided q' expansion,
// per-head V projection) and the fused decode stay hand-written (tc_gemm.cu,
// el_decode_tc.cu).
//
// Row-major C[M][N] = A[M][K] . B[N][K]^T + bias[N]  ==  column-major
// C'[N x M] = B'^T (N x K) . A' (K x M), bias over the N rows of C'.
#include <cublasLt.h>

#include <map>
#include <mutex>
#include <tuple>
#include <unordered_map>

#include "common.cuh"
#include "kernels.h"

namespace elattn_gpu {

namespace {

#define ELA_CHECK_LT(expr)                                                                              \
    do {                                                                                                \
        cublasStatus_t _s = (expr);                                                                     \
        if (_s != CUBLAS_STATUS_SUCCESS)                                                                \
            throw ::elattn_gpu::Status{ELATTN_ERR_CUDA, std::string(#expr) + " failed: " + std::to_string(int(_s))}; \
    } while (0)

constexpr size_t kWorkspace = 32u << 20;

struct Plan {
    cublasLtMatmulDesc_t op = nullptr;
    cublasLtMatrixLayout_t a = nullptr, b = nullptr, c = nullptr;
    cublasLtMatmulAlgo_t algo{};
    bool has_bias = false;
};

struct LtState {
    std::mutex mu;
    cublasLtHandle_t handle = nullptr;
    std::map<std::tuple<int, int, int, int64_t, int64_t, int64_t, bool, int, int64_t, int64_t, int64_t, int64_t>, Plan>
        plans;
    std::unordered_map<cudaStream_t, void*> workspace;  // one per stream (kernels use it asynchronously)
};

LtState& state() {
    static LtState s;
    return s;
}

Plan& plan_for(LtState& S, const GemmArgs& g) {
    const bool bias = g.bias != nullptr;
    auto key = std::make_tuple(g.M, g.N, g.K, g.lda, g.ldb, g.ldc, bias, g.Z, g.sAz, g.sBz, g.sCz, g.sbz);
    auto it = S.plans.find(key);
    if (it != S.plans.end()) return it->second;
    Plan p;
    p.has_bias = bias;
    ELA_CHECK_LT(cublasLtMatmulDescCreate(&p.op, CUBLAS_COMPUTE_32F, CUDA_R_32F));
    const cublasOperation_t tA = CUBLAS_OP_T, tB = CUBLAS_OP_N;
    ELA_CHECK_LT(cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_TRANSA, &tA, sizeof(tA)));
    ELA_CHECK_LT(cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_TRANSB, &tB, sizeof(tB)));
    if (bias) {
        const cublasLtEpilogue_t epi = CUBLASLT_EPILOGUE_BIAS;
        const cudaDataType_t bt = CUDA_R_16BF;  // fp32 bias with bf16 D has no algorithm (tools/probes/lt_probe.cu)
        ELA_CHECK_LT(cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_EPILOGUE, &epi, sizeof(epi)));
        ELA_CHECK_LT(cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_BIAS_DATA_TYPE, &bt, sizeof(bt)));
    }
    // lt-A = our B viewed column-major (K x N, ld ldb), transposed; lt-B = our A (K x M, ld lda)
    ELA_CHECK_LT(cublasLtMatrixLayoutCreate(&p.a, CUDA_R_16BF, uint64_t(g.K), uint64_t(g.N), g.ldb));
    ELA_CHECK_LT(cublasLtMatrixLayoutCreate(&p.b, CUDA_R_16BF, uint64_t(g.K), uint64_t(g.M), g.lda));
    ELA_CHECK_LT(cublasLtMatrixLayoutCreate(&p.c, CUDA_R_16BF, uint64_t(g.N), uint64_t(g.M), g.ldc));
    if (g.Z > 1) {  // strided batch: matrix z at base + z * stride (elements)
        const int32_t cnt = g.Z;
        const int64_t sa = g.sBz, sb = g.sAz, sc = g.sCz;
        for (auto [lay, stride] : {std::pair{p.a, sa}, std::pair{p.b, sb}, std::pair{p.c, sc}}) {
            ELA_CHECK_LT(cublasLtMatrixLayoutSetAttribute(lay, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &cnt, sizeof(cnt)));
            ELA_CHECK_LT(cublasLtMatrixLayoutSetAttribute(lay, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &stride,
                                                          sizeof(stride)));
        }
        if (bias) {
            const int64_t bs = g.sbz;
            ELA_CHECK_LT(cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_BIAS_BATCH_STRIDE, &bs, sizeof(bs)));
        }
    }
    cublasLtMatmulPreference_t pref;
    ELA_CHECK_LT(cublasLtMatmulPreferenceCreate(&pref));
    const size_t ws = kWorkspace;
    ELA_CHECK_LT(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &ws, sizeof(ws)));
    cublasLtMatmulHeuristicResult_t res{};
    int found = 0;
    const cublasStatus_t hs = cublasLtMatmulAlgoGetHeuristic(S.handle, p.op, p.a, p.b, p.c, p.c, pref, 1, &res, &found);
    cublasLtMatmulPreferenceDestroy(pref);
    ELA_REQUIRE(hs == CUBLAS_STATUS_SUCCESS && found > 0, ELATTN_ERR_UNSUPPORTED, "cuBLASLt: no algorithm");
    p.algo = res.algo;
    return S.plans.emplace(key, p).first->second;
}

}  // namespace

bool lt_gemm_supported(const GemmArgs& g) {
    return g.Z >= 1 && (g.bias == nullptr || g.bias16 != nullptr) && g.M > 0 && g.N > 0 && g.K > 0 && g.lda % 8 == 0 && g.ldb % 8 == 0 && g.ldc % 8 == 0;
}

void launch_lt_gemm(const GemmArgs& g, cudaStream_t st) {
    LtState& S = state();
    std::lock_guard<std::mutex> lock(S.mu);
    if (!S.handle) ELA_CHECK_LT(cublasLtCreate(&S.handle));
    void*& ws = S.workspace[st];
    if (!ws) ELA_CHECK_CUDA(cudaMalloc(&ws, kWorkspace));
    Plan& p = plan_for(S, g);
    if (p.has_bias)
        ELA_CHECK_LT(cublasLtMatmulDescSetAttribute(p.op, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &g.bias16, sizeof(g.bias16)));
    const float alpha = g.alpha, beta = 0.f;
    ELA_CHECK_LT(cublasLtMatmul(S.handle, p.op, &alpha, g.B, p.a, g.A, p.b, &beta, g.C, p.c, g.C, p.c, &p.algo, ws,
                                kWorkspace, st));
}

void release_lt_stream(cudaStream_t st) {
    LtState& S = state();
    std::lock_guard<std::mutex> lock(S.mu);
    auto it = S.workspace.find(st);
    if (it == S.workspace.end()) return;
    if (it->second) cudaFree(it->second);
    S.workspace.erase(it);
}

}  // namespace elattn_gpu
