// gemm.cu — K5 GEMM dispatch. Stage 1: cuBLAS (library GEMM) so the whole
// forward step is correct end to end; the hand-written tcgen05/TMEM kernel
// (gemm_tc.cu) replaces it shape by shape once it is parity-green against this.
#include <cublas_v2.h>

#include "gemm.h"

namespace ppdk {

struct GemmContext {
  cublasHandle_t handle = nullptr;
};

GemmContext* gemm_create() {
  GemmContext* c = new GemmContext();
  if (cublasCreate(&c->handle) != CUBLAS_STATUS_SUCCESS) {
    delete c;
    return nullptr;
  }
  cublasSetMathMode(c->handle, CUBLAS_DEFAULT_MATH);
  return c;
}

void gemm_destroy(GemmContext* c) {
  if (!c) return;
  if (c->handle) cublasDestroy(c->handle);
  delete c;
}

cudaError_t gemm_run(GemmContext* c, const __nv_bfloat16* A, const __nv_bfloat16* B, void* C, int M,
                     int N, int K, bool out_f32, cudaStream_t s) {
  if (M == 0) return cudaSuccess;
  cublasSetStream(c->handle, s);
  const float alpha = 1.f, beta = 0.f;
  // row-major C[M][N] = A B^T  <=>  column-major C^T[N][M] = B^T(op T of [K][N]) . A
  cublasStatus_t st = cublasGemmEx(c->handle, CUBLAS_OP_T, CUBLAS_OP_N, N, M, K, &alpha, B,
                                   CUDA_R_16BF, K, A, CUDA_R_16BF, K, &beta, C,
                                   out_f32 ? CUDA_R_32F : CUDA_R_16BF, N, CUBLAS_COMPUTE_32F,
                                   CUBLAS_GEMM_DEFAULT);
  return st == CUBLAS_STATUS_SUCCESS ? cudaSuccess : cudaErrorUnknown;
}

}  // namespace ppdk
