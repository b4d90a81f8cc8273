// Probe: does cuBLASLt offer fp32 (TF32 compute) matmuls with the
// RELU_AUX_BIAS / DRELU_BGRAD / BIAS epilogues on this GPU?
#include <cublasLt.h>
#include <cstdio>
int main() {
    cublasLtHandle_t h; cublasLtCreate(&h);
    const int m = 512, n = 2048, k = 368;
    void* ws; cudaMalloc(&ws, 32 << 20);
    float *A, *B, *C, *bias; void* aux;
    cudaMalloc(&A, sizeof(float) * m * k); cudaMalloc(&B, sizeof(float) * k * n); cudaMalloc(&C, sizeof(float) * m * n);
    cudaMalloc(&bias, sizeof(float) * m); cudaMalloc(&aux, m * n / 8 + 1024);
    cublasLtEpilogue_t eps[] = {CUBLASLT_EPILOGUE_DEFAULT, CUBLASLT_EPILOGUE_RELU_BIAS, CUBLASLT_EPILOGUE_RELU_AUX_BIAS,
                                CUBLASLT_EPILOGUE_DRELU_BGRAD, CUBLASLT_EPILOGUE_DRELU, CUBLASLT_EPILOGUE_BGRADB};
    const char* names[] = {"DEFAULT", "RELU_BIAS", "RELU_AUX_BIAS", "DRELU_BGRAD", "DRELU", "BGRADB"};
    for (int ct = 0; ct < 2; ct++) {
        cublasComputeType_t comp = ct ? CUBLAS_COMPUTE_32F_FAST_TF32 : CUBLAS_COMPUTE_32F;
        for (int e = 0; e < 6; e++) {
            cublasLtMatmulDesc_t op; cublasLtMatmulDescCreate(&op, comp, CUDA_R_32F);
            cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
            cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta));
            cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb));
            cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_EPILOGUE, &eps[e], sizeof(eps[e]));
            cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &bias, sizeof(bias));
            int64_t ld = (m + 127) / 128 * 128;
            cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_EPILOGUE_AUX_POINTER, &aux, sizeof(aux));
            cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_EPILOGUE_AUX_LD, &ld, sizeof(ld));
            cublasLtMatrixLayout_t la, lb, lc;
            cublasLtMatrixLayoutCreate(&la, CUDA_R_32F, k, m, k);
            cublasLtMatrixLayoutCreate(&lb, CUDA_R_32F, k, n, k);
            cublasLtMatrixLayoutCreate(&lc, CUDA_R_32F, m, n, m);
            cublasLtMatmulPreference_t pref; cublasLtMatmulPreferenceCreate(&pref);
            size_t wsz = 32 << 20;
            cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsz, sizeof(wsz));
            cublasLtMatmulHeuristicResult_t res[4]; int got = 0;
            cublasStatus_t s = cublasLtMatmulAlgoGetHeuristic(h, op, la, lb, lc, lc, pref, 4, res, &got);
            float t = -1;
            if (s == CUBLAS_STATUS_SUCCESS && got > 0) {
                float one = 1, zero = 0;
                cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
                for (int w = 0; w < 3; w++) cublasLtMatmul(h, op, &one, A, la, B, lb, &zero, C, lc, C, lc, &res[0].algo, ws, wsz, 0);
                cudaEventRecord(e0);
                for (int r = 0; r < 20; r++) cublasLtMatmul(h, op, &one, A, la, B, lb, &zero, C, lc, C, lc, &res[0].algo, ws, wsz, 0);
                cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&t, e0, e1); t = t / 20 * 1e3;
            }
            printf("%s %-14s status=%d algos=%d  %.2f us  (%s)\n", ct ? "tf32" : "fp32", names[e], (int)s, got, t,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
