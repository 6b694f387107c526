// Which cuBLASLt configurations have an algorithm for C[M][N] (bf16) = A[M][K] B[N][K]^T + bias?
#include <cublasLt.h>
#include <cstdio>
int main() {
    cublasLtHandle_t h; cublasLtCreate(&h);
    const int M = 1280, N = 1024, K = 1024;
    for (int variant = 0; variant < 4; ++variant) {
        cublasLtMatmulDesc_t op; cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F, CUDA_R_32F);
        cublasOperation_t tA = CUBLAS_OP_T, tB = CUBLAS_OP_N;
        cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &tA, sizeof(tA));
        cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &tB, sizeof(tB));
        if (variant >= 1) {
            cublasLtEpilogue_t e = CUBLASLT_EPILOGUE_BIAS;
            cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_EPILOGUE, &e, sizeof(e));
        }
        if (variant == 2) { cudaDataType_t bt = CUDA_R_32F; cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_BIAS_DATA_TYPE, &bt, sizeof(bt)); }
        if (variant == 3) { cudaDataType_t bt = CUDA_R_16BF; cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_BIAS_DATA_TYPE, &bt, sizeof(bt)); }
        cublasLtMatrixLayout_t a, b, c;
        cublasLtMatrixLayoutCreate(&a, CUDA_R_16BF, K, N, K);
        cublasLtMatrixLayoutCreate(&b, CUDA_R_16BF, K, M, K);
        cublasLtMatrixLayoutCreate(&c, CUDA_R_16BF, N, M, N);
        cublasLtMatmulPreference_t pref; cublasLtMatmulPreferenceCreate(&pref);
        size_t ws = 32u << 20;
        cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &ws, sizeof(ws));
        cublasLtMatmulHeuristicResult_t r[4]; int found = 0;
        cublasStatus_t s = cublasLtMatmulAlgoGetHeuristic(h, op, a, b, c, c, pref, 4, r, &found);
        printf("variant %d (0 none, 1 bias default, 2 bias f32, 3 bias bf16): status %d found %d\n", variant, int(s), found);
    }
    return 0;
}
