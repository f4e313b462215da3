// kernels.h — host-visible declarations of the device kernels' launchers.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "gemm_tc.h"

namespace ppdk {

typedef __nv_bfloat16 bf16;

// One attention work item (a CTA per item per kv head).
struct AttnItem {
  int kind;       // 0 decode, 1 prefill tile
  int seq;        // sequence index in the step
  int q_tok0;     // first query token (within the sequence's new tokens)
  int n_q;        // query tokens in this tile (decode: 1)
  int key_begin;  // decode split: key range
  int key_end;
  int split;      // split index, n_splits total; ws_index = workspace slot
  int n_splits;
  int ws_index;
  int pad[3];
};

struct AttnParams {
  const AttnItem* items;
  const bf16* q;             // [total_q][Hq][Dh]
  bf16* out;                 // [total_q][Hq][Dh]
  const int* q_start;        // [n_seqs+1]
  const int* ctx;            // [n_seqs]
  const int* block_tables;   // [n_seqs][max_blocks]
  int max_blocks;
  int n_layers, layer, n_q_heads, n_kv_heads, group;
  float scale_log2;
  float* ws_o;               // split partials [slot][Hkv][G][Dh]
  float* ws_ml;              // [slot][Hkv][G][2]
  int* counters;             // [n_seqs][Hkv], zero-initialised, self-resetting
  // balanced decode schedule: CTA c owns decode segments [seg_start[c], seg_start[c+1])
  const int* seg_start;
  int* mix_ctr;              // K2 queue heads + done counter [3], zero-initialised, self-resetting
  int overlap;               // decode: stream cached K/V before waiting on the predecessor (pdl_overlap)
  int l2_hint;               // decode: K/V TMA loads carry an L2 evict-first policy
};

// Persistent decode attention over balanced key segments (kv head in item.pad[0]).
cudaError_t launch_decode_attention(const void* kv_map, const AttnParams& p, int n_cta, int group,
                                    cudaStream_t stream);

int make_kv_tensor_map(void* map_out /* CUtensorMap, 128 B */, const void* pool, uint64_t total_rows);
cudaError_t launch_paged_attention(const void* kv_map, const AttnParams& p, int n_items,
                                   cudaStream_t stream);
// K2 fused mixed step, one persistent launch of 148 CTAs pulling from two
// queues: n_pf_tiles = (prefill items at pf_items) x n_kv_heads tcgen05 tiles
// (n_pf CTAs start there) and the balanced decode schedule's n_vcta virtual
// CTAs (two decode instances per CTA)
cudaError_t launch_mixed_attention(const void* kv_map, const AttnParams& p, const AttnItem* pf_items, int n_pf,
                                   int n_pf_tiles, int n_vcta, cudaStream_t stream);
// persistent tcgen05 prefill: min(148, tiles) CTAs over an atomic tile queue
// (items longest first; queue head / done counter in p.mix_ctr)
cudaError_t launch_prefill_attention_persistent(const void* kv_map, const AttnParams& p, const AttnItem* items,
                                                int n_items, cudaStream_t stream);
// tcgen05/TMEM prefill tiles (kind 1 items of 128/G tokens)
cudaError_t launch_prefill_attention_tc(const void* kv_map, const AttnParams& p, int n_items, cudaStream_t stream);

// RoPE + paged KV write: everything one token row needs (ops_dev.cuh rope_kv_unit)
struct RopeArgs {
  const float* qkv;  // fp32 partial slices [T][qd + 2kd]
  GemmParts parts;
  const float* bias;
  const int *row_seq, *row_pos, *block_tables;
  int max_blocks;
  const float *rope_cos, *rope_sin;
  bf16 *q_out, *kv;
  int Hq, Hkv, Dh, n_layers, layer, block_tokens;
};

// ---- K8 decode layer kernel (layer_tc.cu) ----
// One persistent launch per layer for steps of <= 256 token rows: o-proj ->
// residual add + RMSNorm -> gate|up -> SiLU -> down -> residual add + RMSNorm
// -> the NEXT layer's qkv -> RoPE + KV write. Each GEMM ("job") is a stream-K
// partition of its (weight tile, k-block) items over the CTAs; the glue
// between jobs runs after a grid-wide counter barrier, while the TMA producer
// keeps streaming the next job's weights (they do not depend on the glue).
constexpr int kLayerMaxJobs = 4;
struct LayerJob {
  float* out;       // fp32 K-partial slices, slice j at out + j * parts.stride
  int N, K, kbt;    // output columns, reduction length, 64-wide k-blocks per weight tile
  long long total;  // weight tiles * kbt items
  int ts;           // CTAs sharing the items: CTA c < ts owns [c*total/ts, (c+1)*total/ts)
  GemmParts parts;  // slice rule the glue reads `out` with
};
struct LayerParams {
  alignas(64) uint8_t map_w[kLayerMaxJobs][128];  // CUtensorMap of each job's weights
  alignas(64) uint8_t map_x[kLayerMaxJobs][128];  // ... and of its activations
  LayerJob job[kLayerMaxJobs];
  int n_jobs, T, bn, stages, stage_bytes, n_cta;
  int l2_ahead;    // weight k-blocks the producer prefetches into L2 beyond the ring while waiting
  unsigned* sync;  // [n_jobs][2] epilogue-done / glue-done counters, zeroed per step
  bf16 *x, *h, *m;
  const bf16* norm_w;
  float eps;
  int d_model, F;
  RopeArgs rope;  // the next layer's RoPE + KV write (job 3)
};
// grid-wide layout of a job for T token rows; false if its partial slices
// would not fit `max_slices` workspace slices
bool layer_plan_job(LayerJob& j, float* out, int T, int N, int K, int n_cta, int max_slices);
// smem ring for T token rows (0 stages: T too large)
void layer_shape(int T, int* bn, int* stages, int* stage_bytes, int* smem);
cudaError_t launch_decode_layer(const LayerParams& p, int smem, cudaStream_t s);

// ---- small fused ops (ops.cu) ----
cudaError_t launch_fill_random(bf16* dst, uint64_t n, uint64_t seed, int tensor, int layer,
                               cudaStream_t s);
// fused QKV weight [Hq*Dh + 2*Hkv*Dh][d]: rows < qd from tensor WQ, then WK, then WV
cudaError_t launch_fill_qkv(bf16* dst, int qd, int kd, int d, uint64_t seed, int layer, cudaStream_t s);
// weight matrix [N][K], row-major
cudaError_t launch_fill_matrix(bf16* dst, uint64_t N, uint64_t K, uint64_t seed, int tensor, int layer,
                               cudaStream_t s);
cudaError_t launch_fill_bias(float* dst, int qd, int kd, uint64_t seed, int layer, cudaStream_t s);
// gate/up weight [2F][d], interleaved in groups of 64 rows: rows [128j, 128j+64) = gate
// rows [64j, 64j+64), rows [128j+64, 128j+128) = up rows [64j, 64j+64)
cudaError_t launch_fill_gate_up(bf16* dst, int F, int d, uint64_t seed, int layer, cudaStream_t s);
cudaError_t launch_fill_const(bf16* dst, uint64_t n, float v, cudaStream_t s);

cudaError_t launch_embed(const int* tokens, const bf16* embed, bf16* x, int T, int d, cudaStream_t s);
// x = rbf(x + rbf(delta)) (if delta); h = rbf(rmsnorm(x) * w). delta may be fp32 split partials
// (the valid slices of `parts`, summed in slice order first), or bf16 when delta_bf16 != null.
cudaError_t launch_add_rmsnorm(bf16* x, const float* delta_f32, const GemmParts& parts, const bf16* delta_bf16,
                               const bf16* w, bf16* h, int T, int d, float eps, cudaStream_t s);
// final: for each selected row r = rows[i]: v = x[r] (+ delta[r]); out[i] = rbf(rmsnorm(v) * w)
cudaError_t launch_final_norm(const bf16* x, const float* delta_f32, const GemmParts& parts,
                              const bf16* delta_bf16, const int* rows, int n_rows, const bf16* w,
                              bf16* out, int T, int d, float eps, cudaStream_t s);
// qkv fp32 [T][qd+2kd] (+bias) -> q bf16 [T][Hq][Dh] roped; k roped, v -> paged pool
cudaError_t launch_rope_kv_write(const float* qkv, const GemmParts& parts, const float* bias, const int* row_seq,
                                 const int* row_pos, const int* block_tables, int max_blocks,
                                 const float* rope_cos, const float* rope_sin, bf16* q_out,
                                 bf16* kv_pool, int T, int Hq, int Hkv, int Dh, int n_layers,
                                 int layer, int block_tokens, cudaStream_t s);
// gate/up fp32 [T][2F] interleaved (see launch_fill_gate_up) -> m = rbf(silu(g) * u) [T][F]
cudaError_t launch_silu_mul(const float* gu, const GemmParts& parts, bf16* m, int T, int F, cudaStream_t s);
cudaError_t launch_argmax(const float* logits, int n, int V, int* out, cudaStream_t s);
cudaError_t launch_f32_to_bf16(const float* in, bf16* out, uint64_t n, cudaStream_t s);

// ---- KV transfer (kv_copy.cu) ----
struct KvCopyParams {
  const bf16* src_pool;
  bf16* dst_pool;
  const int* src_blocks;  // block table rows (device)
  const int* dst_blocks;
  int start, n_tokens;
  int n_layers, n_kv_heads, block_tokens, head_dim;
};
cudaError_t launch_kv_copy(const KvCopyParams& p, cudaStream_t s);
cudaError_t launch_pull_copy(const uint4* src, uint4* dst, long n16, cudaStream_t s);

}  // namespace ppdk

namespace ppdk {
// Launch with the programmatic-stream-serialization attribute (PDL) so the
// kernel may begin while its predecessor drains; kernels call pdl_wait()
// before consuming predecessor outputs.
bool pdl_enabled();
// light kernels trigger their successor before waiting (tuning "pdl_overlap",
// default off: measured 2.5% slower): see pdl_enter in common.cuh
int pdl_overlap();
void set_pdl_overlap(int on);
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
// same, as clusters of `cluster_x` CTAs (grid.x must be a multiple)
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_cluster(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, int cluster_x,
                               cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster_x;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
}  // namespace ppdk
