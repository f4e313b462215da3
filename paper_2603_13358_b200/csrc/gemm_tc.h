// gemm_tc.h — tcgen05 GEMM launcher (gemm_tc.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stddef.h>

namespace ppdk {

typedef __nv_bfloat16 bf16;

struct GemmTcParams {
  void* out;
  int T, N, K, ldo, bn, bn_cols, out_f32, splits, stages, tmem_cols;
  size_t split_stride;  // floats between split partial slices
};

// out[T][N] (+ split slices) = X[T][K] . W[N][K]^T ; splits > 1 needs out_f32
cudaError_t gemm_tc_run(const bf16* X, const bf16* W, void* out, int T, int N, int K, bool out_f32, int splits,
                        size_t split_stride, cudaStream_t s);
// K-split count that fills the 148 SMs for this shape (1 when the tile grid already does)
int gemm_tc_plan_splits(int T, int N, int K);

}  // namespace ppdk
