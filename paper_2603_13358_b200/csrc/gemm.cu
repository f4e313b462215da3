// gemm.cu — K5 GEMM entry points of the forward step: the tcgen05 kernel
// (gemm_tc.cu) is the only product path. cuBLAS appears here solely as the
// library reference ppd_op_gemm exposes to the parity tests.
#include <cublas_v2.h>

#include <cstdlib>
#include <cstring>

#include "gemm.h"
#include "gemm_tc.h"
#include "kernels.h"

namespace ppdk {

struct GemmContext {
  cublasHandle_t handle = nullptr;  // ppd_op_gemm (test reference) only
};

GemmContext* gemm_create() {
  GemmContext* c = new GemmContext();
  if (cublasCreate(&c->handle) != CUBLAS_STATUS_SUCCESS) {
    delete c;
    return nullptr;
  }
  return c;
}

void gemm_destroy(GemmContext* c) {
  if (!c) return;
  if (c->handle) cublasDestroy(c->handle);
  delete c;
}

cudaError_t gemm_run_cublas(GemmContext* c, const __nv_bfloat16* A, const __nv_bfloat16* B, void* C, int M, int N,
                            int K, bool out_f32, cudaStream_t s) {
  if (M == 0) return cudaSuccess;
  cublasSetStream(c->handle, s);
  const float alpha = 1.f, beta = 0.f;
  // row-major C[M][N] = A B^T  <=>  column-major C^T[N][M] = B^T(op T of [K][N]) . A
  cublasStatus_t st = cublasGemmEx(c->handle, CUBLAS_OP_T, CUBLAS_OP_N, N, M, K, &alpha, B, CUDA_R_16BF, K, A,
                                   CUDA_R_16BF, K, &beta, C, out_f32 ? CUDA_R_32F : CUDA_R_16BF, N,
                                   CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
  return st == CUBLAS_STATUS_SUCCESS ? cudaSuccess : cudaErrorUnknown;
}

cudaError_t gemm_run(const __nv_bfloat16* A, const __nv_bfloat16* B, void* C, int M, int N, int K, bool out_f32,
                     cudaStream_t s) {
  return gemm_tc_run(A, B, C, M, N, K, out_f32, 1, 0, s);
}

cudaError_t gemm_run_split(const __nv_bfloat16* A, const __nv_bfloat16* B, float* C, int M, int N, int K,
                           int max_slices, GemmParts* parts, cudaStream_t s) {
  return gemm_tc_run_parts(A, B, C, M, N, K, max_slices, (size_t)M * N, parts, s);
}

cudaError_t gemm_run_silu(const __nv_bfloat16* A, const __nv_bfloat16* B, __nv_bfloat16* m, int M, int N, int K,
                          cudaStream_t s) {
  if (M == 0) return cudaSuccess;
  return gemm_tc_run_silu(A, B, m, M, N, K, s);
}

}  // namespace ppdk
