// gemm_tc.h — tcgen05 GEMM launcher (gemm_tc.cu) and the description of how
// its fp32 output is spread over K-partial slices (read by the consumers).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stddef.h>

namespace ppdk {

typedef __nv_bfloat16 bf16;

// How a GEMM's fp32 output C[T][N] is stored as partial slices
// out + j*stride, j < n; C = sum of the slices that are VALID for the element.
//  * uniform split (kbt == 0): every slice is valid everywhere.
//  * balanced (stream-K) partition: tiles [0, dp) are whole-K units (one
//    valid slice); the flattened (tile - dp, k-block) space of the other
//    tiles, `total` = (tiles - dp)*kbt items, is cut into `slots` equal
//    contiguous ranges; the j-th range touching a tile writes slice j, so a
//    tile has (owner(last item) - owner(first item) + 1) valid slices.
// Slices are summed in order j = 0, 1, ... (fixed order: deterministic).
struct GemmParts {
  int n = 1;            // slices
  size_t stride = 0;    // floats between slices
  int kbt = 0;          // k-blocks per tile (0 = uniform split)
  int slots = 1;        // ranges (persistent CTAs / pairs)
  int rows = 128;       // weight rows (output columns) per tile
  int bn = 256;         // token rows per tile (a unit: all token sub-tiles of one weight stage)
  int n_tiles_t = 1;    // token tiles
  long long total = 1;  // (tiles - dp) * kbt
  int dp = 0;           // leading whole-K (data-parallel) tiles

  __host__ __device__ __forceinline__ int owner(long long x) const {
    // 32-bit division when the product fits (every shape this library plans:
    // tiles * k-blocks * slots < 2^31); the consumers call this per element
    // group, where a 64-bit division made the small ops instruction-bound
    if ((total + 1) * (long long)slots < (1LL << 31))
      return (int)(((unsigned)(x + 1) * (unsigned)slots + (unsigned)total - 1u) / (unsigned)total) - 1;
    return (int)(((x + 1) * slots + total - 1) / total) - 1;
  }
  // valid slices for output column `col` of token row `tok`
  __host__ __device__ __forceinline__ int valid(int col, int tok) const {
    if (kbt == 0) return n;
    const long long t = (long long)(col / rows) * n_tiles_t + tok / bn - dp;
    if (t < 0) return 1;
    return owner(t * kbt + kbt - 1) - owner(t * kbt) + 1;
  }
};

struct GemmTcParams {
  void* out;
  int T, N, K, ldo, bn, bn_cols, out_f32, splits, stages, tmem_cols;
  size_t split_stride;  // floats between split partial slices
  int balanced;         // 1: stream-K ranges (GemmParts), 0: units of uniform K splits
  int slots;            // persistent CTAs (pairs) the schedule is cut for
  long long total;      // tiles * k-blocks per tile (balanced)
  int epi;              // 0: write C (fp32 slices / bf16); 1: fused SiLU(gate)*up -> bf16 [T][N/2]
  int n_sub;            // token sub-tiles (of bn rows) per unit: every weight stage feeds n_sub MMAs
  int dp;               // balanced: leading whole-K tiles dealt round-robin
  int tail_slots;       // balanced: slots sharing the stream-K tail (<= slots)
  int l2_pre;           // weight k-blocks beyond the smem ring prefetched into L2 before the PDL wait
  int overlap;          // 1: trigger the successor only after our own PDL wait (see pdl_enter)
  int epi_pipe;         // 1: plain epilogue double-buffers its TMEM loads (gemm_tc_set_epi_pipe)
  int l2_hint;          // 1: weight TMA loads carry an L2 evict-first policy
};

// out[T][N] (+ split slices) = X[T][K] . W[N][K]^T ; splits > 1 needs out_f32
cudaError_t gemm_tc_run(const bf16* X, const bf16* W, void* out, int T, int N, int K, bool out_f32, int splits,
                        size_t split_stride, cudaStream_t s);
// fp32 output into partial slices chosen by the planner (uniform split or a
// balanced partition), at most `max_slices` slices of split_stride floats.
cudaError_t gemm_tc_run_parts(const bf16* X, const bf16* W, float* out, int T, int N, int K, int max_slices,
                              size_t split_stride, GemmParts* parts, cudaStream_t s);
// m[T][N/2] = rbf(silu(gate) * up) for the interleaved gate|up weight [N][K]
// (64-row groups, launch_fill_gate_up): the MLP up-projection with SiLU fused
// into the epilogue (no K split; no fp32 round trip through HBM).
cudaError_t gemm_tc_run_silu(const bf16* X, const bf16* W, bf16* m, int T, int N, int K, cudaStream_t s);
// pair_mode: -1 auto, 0 single-CTA kernel, 1 CTA-pair kernel; stage_cap 0 = no cap;
// sched: -1 auto, 0 uniform K split, 1 balanced partition
void gemm_tc_set_tuning(int pair_mode, int stage_cap, int sched);
// T in (256, 512] token rows: one unit per weight tile covering 2 token
// sub-tiles (default on) vs separate 256-row token tiles (A/B knob)
void gemm_tc_set_multi_sub(int mode);
void gemm_tc_set_epi_pipe(bool on);
// L2 evict-first on streamed-once loads: bit 0 GEMM weights, bit 1 decode K/V
void gemm_tc_set_l2_hint(int mask);
int gemm_tc_l2_hint();
// T > 256 rows in separate token tiles: equal tiles (default) vs 256-row tiles (A/B knob)
void gemm_tc_set_even_tiles(bool on);
// two co-resident CTAs per SM (half-depth rings, one accumulator each):
// -1 auto (small token counts), 0 off, 1 whenever the shape allows
void gemm_tc_set_occ2(int mode);
// weight k-blocks each CTA prefetches into L2 (beyond its smem ring) while its
// predecessor finishes: -1 auto, 0 off, n
void gemm_tc_set_l2_pre(int n);
// 2-D TMA map (128 B) of a K-major bf16 [rows][K] matrix, box = box_rows x 64 K
// elements, 128 B swizzle (the layout every tcgen05 kernel here consumes)
bool gemm_tc_map(void* map_out, const void* ptr, int rows, int K, int box_rows);
// K-split count that fills the 148 SMs for this shape (1 when the tile grid already does)
int gemm_tc_plan_splits(int T, int N, int K);

}  // namespace ppdk
