// gemm.h — K5 projection / MLP / lm_head GEMMs: C[M][N] = A[M][K] . B[N][K]^T,
// bf16 operands, fp32 accumulate, fp32 or bf16 output.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace ppdk {
struct GemmContext;
GemmContext* gemm_create();
void gemm_destroy(GemmContext* ctx);
cudaError_t gemm_run(GemmContext* ctx, const __nv_bfloat16* A, const __nv_bfloat16* B, void* C,
                     int M, int N, int K, bool out_f32, cudaStream_t s);
}  // namespace ppdk
