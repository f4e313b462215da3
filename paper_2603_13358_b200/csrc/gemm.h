// gemm.h — K5 projection / MLP / lm_head GEMMs: C[M][N] = A[M][K] . B[N][K]^T,
// bf16 operands, fp32 accumulate, always the hand-written tcgen05 kernel
// (gemm_tc.cu). The cuBLAS context exists only for ppd_op_gemm (test reference).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stddef.h>

#include "gemm_tc.h"

namespace ppdk {
struct GemmContext;
GemmContext* gemm_create();
void gemm_destroy(GemmContext* ctx);
// single-slice product (no K split)
cudaError_t gemm_run(const __nv_bfloat16* A, const __nv_bfloat16* B, void* C, int M, int N, int K, bool out_f32,
                     cudaStream_t s);
// fp32 product written as K-partial slices of M*N floats each (at most
// max_slices; *parts says which slices are valid where, the consumer sums
// them); the planner picks the split / balanced partition that fills the SMs.
cudaError_t gemm_run_split(const __nv_bfloat16* A, const __nv_bfloat16* B, float* C, int M, int N, int K,
                           int max_slices, GemmParts* parts, cudaStream_t s);
// MLP up-projection with SiLU fused: m[M][N/2] = rbf(silu(gate) * up) for the
// interleaved gate|up weight B [N][K].
cudaError_t gemm_run_silu(const __nv_bfloat16* A, const __nv_bfloat16* B, __nv_bfloat16* m, int M, int N, int K,
                          cudaStream_t s);
cudaError_t gemm_run_cublas(GemmContext* ctx, const __nv_bfloat16* A, const __nv_bfloat16* B, void* C, int M,
                            int N, int K, bool out_f32, cudaStream_t s);
}  // namespace ppdk
