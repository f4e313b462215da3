// attention_tc.cu — K3/K4: full- and append-prefill attention over the paged
// KV pool on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// Replaces append_prefill_time / full_prefill_time (reference
// costmodel.cpp:318-331, called simulator.cpp:327-329) for the attention part
// of a prefill chunk. One CTA = 128 query rows (128/G tokens x the G query
// heads of one kv head) of one sequence, causal over the paged history.
//
//   warp 0  K TMA producer, warp 3 V TMA producer: per 128-key block, 8 paged
//           16-token blocks (2-D tensor map over the pool, 128 B swizzle, 16
//           boxes issued lane-parallel) -> 2-stage K and V rings
//   warp 1  MMA issuer (one thread): S_j = Q K_j^T into TMEM (double-buffered),
//           then O += P_{j-1} V_{j-1} with A = P_{j-1} read from TMEM (written
//           over S_{j-1}'s columns) and B = V (MN-major, shared memory)
//   warp 2  TMEM allocator (512 columns: S0 | S1 | O | max exchange)
//   warps 4.. kSW softmax warps, kSW / 4 threads per query row: online
//           softmax on the S row part read with tcgen05.ld, running max
//           agreed through TMEM + a named barrier, exp2 split between MUFU and
//           an f32x2 polynomial, lazy O rescaling (only when the running max
//           grows by more than 2^8), P (bf16) back to TMEM with tcgen05.st,
//           epilogue O / l -> bf16.
#include <cuda.h>

#include "attention_tc_body.cuh"
#include "kernels.h"

namespace ppdk {

#ifndef PPD_PF_SW
constexpr int kSW = 8;  // softmax warps of the standalone kernels: 2 threads per query row (16: 4, measured ~5% slower)
#else
constexpr int kSW = PPD_PF_SW;
#endif
constexpr int kPfThreads = pftc::threads_for(kSW);

__global__ void __launch_bounds__(kPfThreads, 1)
    prefill_attention_tc_kernel(const __grid_constant__ CUtensorMap kv_map, AttnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const pftc::Smem S(smem);
  pdl_wait();
  const AttnItem it = p.items[blockIdx.x];
  if (it.kind != 1) return;  // decode rows are served by the decode kernels
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) pftc::init_barriers<kSW>(S, false);
  if (warp == 2) tc::alloc(S.tmem_slot, pftc::kTmemCols);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *S.tmem_slot;
  pftc::tile<kSW>(&kv_map, p, S, it, blockIdx.y, tmem, warp, lane, true);
  tc::fence_before();
  __syncthreads();
  if (warp == 2) tc::dealloc(tmem, pftc::kTmemCols);
}

// Pure prefill steps: min(148, tiles) persistent CTAs pull the tiles (longest
// first) from an atomic queue, so a chunk's 2-3 waves of uneven causal tiles
// leave no idle SMs at the tail.
__global__ void __launch_bounds__(kPfThreads, 1)
    prefill_attention_persistent_kernel(const __grid_constant__ CUtensorMap kv_map, AttnParams p,
                                        const AttnItem* items, int n_tiles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ int s_next;
  pdl_wait();
  pftc::tile_queue<kSW>(&kv_map, p, smem, items, n_tiles, threadIdx.x >> 5, threadIdx.x & 31, 1, p.mix_ctr,
                   p.mix_ctr + 1, gridDim.x, &s_next);
  pdl_trigger();
}

cudaError_t launch_prefill_attention_persistent(const void* kv_map, const AttnParams& p, const AttnItem* items,
                                                int n_items, cudaStream_t stream) {
  static unsigned long long attr_devs = 0;
  if (first_on_device(&attr_devs)) {
    cudaFuncSetAttribute(prefill_attention_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         pftc::kSmem);
  }
  const int n_tiles = n_items * p.n_kv_heads;
  if (n_tiles == 0) return cudaSuccess;
  if (!p.mix_ctr) return cudaErrorInvalidValue;
  const int grid = n_tiles < device_sms() ? n_tiles : device_sms();
  return launch_pdl(prefill_attention_persistent_kernel, dim3(grid), dim3(kPfThreads), pftc::kSmem, stream,
                    *reinterpret_cast<const CUtensorMap*>(kv_map), p, items, n_tiles);
}

cudaError_t launch_prefill_attention_tc(const void* kv_map, const AttnParams& p, int n_items, cudaStream_t stream) {
  static unsigned long long attr_devs = 0;
  if (first_on_device(&attr_devs)) {
    cudaFuncSetAttribute(prefill_attention_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pftc::kSmem);
  }
  if (n_items == 0) return cudaSuccess;
  dim3 grid(n_items, p.n_kv_heads);
  return launch_pdl(prefill_attention_tc_kernel, grid, dim3(kPfThreads), pftc::kSmem, stream,
                    *reinterpret_cast<const CUtensorMap*>(kv_map), p);
}

}  // namespace ppdk
