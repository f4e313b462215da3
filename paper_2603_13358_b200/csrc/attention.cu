// attention.cu — K1/K2/K3/K4: paged attention over the HBM KV pool, one launch
// for a mixed batch of decode rows and prefill/append query tiles.
//
// Replaces the analytic decode_step_time / append_prefill_time /
// full_prefill_time service times (reference costmodel.cpp:318-379, called at
// simulator.cpp:327-329 and :397) with real attention over the cached KV.
//
// Work items (one CTA each, grid = items x kv_heads):
//   DECODE  one query token of sequence s, keys [key_begin, key_end) of a
//           KV split; the G query heads sharing kv head h are rows 0..G-1 of
//           a 16-row MMA tile; the 4 consumer warps take interleaved 16-key
//           blocks of every 64-key stage and merge at the end (and across
//           splits through a workspace, last CTA merges).
//   PREFILL TQ = 64/G query tokens x G heads = 64 rows (16 per consumer warp),
//           causal over keys [0, ctx + last token of the tile].
// Paged K/V blocks (16 tokens x 128 dims per (block, layer, K|V, kv head)) are
// staged into shared memory by TMA (2-D tensor map over the pool, 128-byte
// swizzle) by a dedicated producer warp through a 3-stage mbarrier ring. The
// QK^T and PV contractions use warp-level mma.sync (bf16 in, fp32 accumulate);
// softmax is online, fp32, with quad shuffles for the row reductions.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "attention_tc_body.cuh"
#include "common.cuh"
#include "kernels.h"

namespace ppdk {

namespace {

constexpr int kBT = 16;          // tokens per KV block
constexpr int kDh = 128;         // head dim
constexpr int kStageBlocks = 4;  // blocks per pipeline stage (64 keys)
constexpr int kStages = 3;
constexpr int kRows = 64;        // query rows per CTA (prefill)
constexpr int kConsumerWarps = 4;
constexpr int kThreads = (kConsumerWarps + 1) * 32;
constexpr int kBlockBytes = kBT * kDh * 2;                       // 4 KB
constexpr int kStageBytes = kStageBlocks * 2 * kBlockBytes;      // 32 KB (K and V)
constexpr int kSmemBytes = 1024 + kStages * kStageBytes + 256;   // 2 CTAs per SM

PPD_DEV void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
PPD_DEV void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
PPD_DEV void mma16816(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// byte offset of (row, dim) inside one 16x128 K/V block laid out by TMA as two
// 2 KB halves (dims 0-63 | 64-127) of 16 rows x 128 B with the 128-byte swizzle
PPD_DEV uint32_t kv_off(int row, int dim) {
  int half = dim >> 6;
  int chunk = (dim & 63) >> 3;
  return half * 2048 + row * 128 + ((chunk ^ (row & 7)) << 4) + ((dim & 7) << 1);
}

PPD_DEV void tma_load_2d(void* smem, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

PPD_DEV void tma_load_2d_hint(void* smem, const CUtensorMap* map, int x, int y, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

}  // namespace

__global__ void __launch_bounds__(kThreads, 2)
    paged_attention_kernel(const __grid_constant__ CUtensorMap kv_map, AttnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stage_base = smem;                                  // kStages * 32 KB
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty_bar = full_bar + kStages;
  int* flag = reinterpret_cast<int*>(empty_bar + kStages);

  pdl_wait();
  const AttnItem it = p.items[blockIdx.x];
  const int kvh = blockIdx.y;
  const int G = p.group;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool is_decode = it.kind == 0;
  const int s = it.seq;
  const int ctx = p.ctx[s];
  const int q_base = p.q_start[s];

  // key range
  int key_begin, key_end;
  if (is_decode) {
    key_begin = it.key_begin;
    key_end = it.key_end;
  } else {
    key_begin = 0;
    key_end = ctx + it.q_tok0 + it.n_q;  // last token of the tile attends up to itself
  }
  const int n_stages_total = (key_end - key_begin + kStageBlocks * kBT - 1) / (kStageBlocks * kBT);
  const int* btab = p.block_tables + (size_t)s * p.max_blocks;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], kConsumerWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ---------------- producer warp: TMA loads of paged K/V ----------------
    if (lane == 0) {
      const int first_blk = key_begin / kBT;
      const int last_blk = (key_end - 1) / kBT;  // inclusive
      for (int st = 0; st < n_stages_total; ++st) {
        int slot = st % kStages;
        if (st >= kStages) mbar_wait(&empty_bar[slot], ((st / kStages) - 1) & 1);
        int b0 = first_blk + st * kStageBlocks;
        int nb = min(kStageBlocks, last_blk - b0 + 1);
        mbar_arrive_expect_tx(&full_bar[slot], nb * 2 * kBlockBytes);
        uint8_t* dst = stage_base + slot * kStageBytes;
        for (int b = 0; b < nb; ++b) {
          int blk = btab[b0 + b];
          // pool row of (blk, layer, K, kvh, token 0)
          int rowK = (((blk * p.n_layers + p.layer) * 2 + 0) * p.n_kv_heads + kvh) * kBT;
          int rowV = rowK + p.n_kv_heads * kBT;
          tma_load_2d(dst + (b * 2 + 0) * kBlockBytes, &kv_map, 0, rowK, &full_bar[slot]);
          tma_load_2d(dst + (b * 2 + 0) * kBlockBytes + 2048, &kv_map, 64, rowK, &full_bar[slot]);
          tma_load_2d(dst + (b * 2 + 1) * kBlockBytes, &kv_map, 0, rowV, &full_bar[slot]);
          tma_load_2d(dst + (b * 2 + 1) * kBlockBytes + 2048, &kv_map, 64, rowV, &full_bar[slot]);
        }
      }
    }
    return;
  }

  // ---------------- consumer warps ----------------
  const int g = lane >> 2, t = lane & 3;
  const int row_base = is_decode ? 0 : warp * 16;
  const float sl2 = p.scale_log2;

  // Q fragments for the 8 k-steps, loaded straight from global (row r of the
  // tile = token r / G, head r % G; rows past the tile are zero)
  uint32_t qa[8][4];
  {
    const int rows = is_decode ? G : (it.n_q * G);
    const uint32_t* qrow[2];
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      int r = row_base + g + hr * 8;
      qrow[hr] = r < rows ? reinterpret_cast<const uint32_t*>(
                                p.q + ((size_t)(q_base + it.q_tok0 + r / G) * p.n_q_heads + kvh * G + r % G) * kDh)
                          : nullptr;
    }
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      int w0 = (kk * 16 + 2 * t) >> 1;  // 32-bit word index of dims (16kk+2t, +1)
      qa[kk][0] = qrow[0] ? __ldg(qrow[0] + w0) : 0u;
      qa[kk][1] = qrow[1] ? __ldg(qrow[1] + w0) : 0u;
      qa[kk][2] = qrow[0] ? __ldg(qrow[0] + w0 + 4) : 0u;
      qa[kk][3] = qrow[1] ? __ldg(qrow[1] + w0 + 4) : 0u;
    }
  }
  // causal limit (position) of this thread's two rows
  int pos_r0, pos_r1;
  {
    int r0 = row_base + g, r1 = row_base + g + 8;
    if (is_decode) {
      pos_r0 = pos_r1 = ctx;
    } else {
      int lim = it.n_q * G;
      pos_r0 = r0 < lim ? ctx + it.q_tok0 + r0 / G : -1;
      pos_r1 = r1 < lim ? ctx + it.q_tok0 + r1 / G : -1;
    }
  }

  float o[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  const int first_blk = key_begin / kBT;
  for (int st = 0; st < n_stages_total; ++st) {
    int slot = st % kStages;
    mbar_wait(&full_bar[slot], (st / kStages) & 1);
    const uint32_t sbase = smem_u32(stage_base + slot * kStageBytes);
    const int stage_key0 = (first_blk + st * kStageBlocks) * kBT;
    // decode: this warp's block within the stage; prefill: all 4 blocks
    const int stage_blocks_valid = min(kStageBlocks, (key_end - 1) / kBT - (first_blk + st * kStageBlocks) + 1);
    const int nblk = is_decode ? 1 : stage_blocks_valid;  // never touch blocks not loaded
    const int blk_lo = is_decode ? warp : 0;
    if (blk_lo < stage_blocks_valid) {
      float sc[8][4];  // up to 8 n-tiles of 8 keys
#pragma unroll
      for (int i = 0; i < 8; ++i) sc[i][0] = sc[i][1] = sc[i][2] = sc[i][3] = 0.f;
#pragma unroll
      for (int bi = 0; bi < kStageBlocks; ++bi) {
        if (bi < nblk) {
          const int b = blk_lo + bi;
          const uint32_t kb = sbase + (b * 2 + 0) * kBlockBytes;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            int krow = (lane & 7) + (lane >> 4) * 8;
            int dim = kk * 16 + ((lane >> 3) & 1) * 8;
            uint32_t b0, b1, b2, b3;
            ldsm_x4(kb + kv_off(krow, dim), b0, b1, b2, b3);
            mma16816(sc[bi * 2 + 0], qa[kk], b0, b1);
            mma16816(sc[bi * 2 + 1], qa[kk], b2, b3);
          }
        }
      }
      // scale + mask, row max
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        if (nt < nblk * 2) {
          int key = stage_key0 + (blk_lo + nt / 2) * kBT + (nt & 1) * 8 + 2 * t;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            int k = key + e;
            bool ok0 = k <= pos_r0 && k >= key_begin && k < key_end;
            bool ok1 = k <= pos_r1 && k >= key_begin && k < key_end;
            sc[nt][e] = ok0 ? sc[nt][e] * sl2 : -INFINITY;
            sc[nt][2 + e] = ok1 ? sc[nt][2 + e] * sl2 : -INFINITY;
            mx0 = fmaxf(mx0, sc[nt][e]);
            mx1 = fmaxf(mx1, sc[nt][2 + e]);
          }
        }
      }
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
      float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
      // rows with nothing valid yet keep -inf; use 0 as the exponent base
      float base0 = mn0 == -INFINITY ? 0.f : mn0;
      float base1 = mn1 == -INFINITY ? 0.f : mn1;
      float corr0 = exp2f(m0 - base0), corr1 = exp2f(m1 - base1);
      m0 = mn0;
      m1 = mn1;
      float rs0 = 0.f, rs1 = 0.f;
      uint32_t pa[4][4];  // P as A fragments, per 16-key block
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        if (nt < nblk * 2) {
          float p0 = exp2f(sc[nt][0] - base0), p1 = exp2f(sc[nt][1] - base0);
          float p2 = exp2f(sc[nt][2] - base1), p3 = exp2f(sc[nt][3] - base1);
          rs0 += p0 + p1;
          rs1 += p2 + p3;
          pa[nt / 2][(nt & 1) * 2 + 0] = pack2(p0, p1);
          pa[nt / 2][(nt & 1) * 2 + 1] = pack2(p2, p3);
        }
      }
      rs0 += __shfl_xor_sync(0xffffffffu, rs0, 1);
      rs0 += __shfl_xor_sync(0xffffffffu, rs0, 2);
      rs1 += __shfl_xor_sync(0xffffffffu, rs1, 1);
      rs1 += __shfl_xor_sync(0xffffffffu, rs1, 2);
      l0 = l0 * corr0 + rs0;
      l1 = l1 * corr1 + rs1;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        o[i][0] *= corr0;
        o[i][1] *= corr0;
        o[i][2] *= corr1;
        o[i][3] *= corr1;
      }
      // O += P V
#pragma unroll
      for (int bi = 0; bi < kStageBlocks; ++bi) {
        if (bi < nblk) {
          const int b = blk_lo + bi;
          const uint32_t vb = sbase + (b * 2 + 1) * kBlockBytes;
          uint32_t a[4] = {pa[bi][0], pa[bi][1], pa[bi][2], pa[bi][3]};
#pragma unroll
          for (int nt = 0; nt < 16; nt += 2) {
            int krow = (lane & 7) + ((lane >> 3) & 1) * 8;
            int dim = nt * 8 + (lane >> 4) * 8;
            uint32_t b0, b1, b2, b3;
            ldsm_x4_t(vb + kv_off(krow, dim), b0, b1, b2, b3);
            mma16816(o[nt], a, b0, b1);
            mma16816(o[nt + 1], a, b2, b3);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[slot]);
  }
  pdl_trigger();

  if (!is_decode) {
    // prefill rows: normalise and store bf16
    const int lim = it.n_q * G;
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      int r = row_base + g + hr * 8;
      if (r >= lim) continue;
      float inv = 1.f / (hr ? l1 : l0);
      int tok = r / G, h = r % G;
      bf16* dst = p.out + ((size_t)(q_base + it.q_tok0 + tok) * p.n_q_heads + kvh * G + h) * kDh;
#pragma unroll
      for (int nt = 0; nt < 16; ++nt) {
        uint32_t v = pack2(o[nt][hr * 2] * inv, o[nt][hr * 2 + 1] * inv);
        *reinterpret_cast<uint32_t*>(dst + nt * 8 + 2 * t) = v;
      }
    }
    return;
  }

  // ---- decode: merge the 4 consumer warps (rows 0..G-1) through shared ----
  // all TMA traffic has been consumed; reuse the stage buffers
  named_barrier_sync(1, kConsumerWarps * 32);
  float* sm_o = reinterpret_cast<float*>(stage_base);           // [4 warps][16 rows][128]
  float* sm_ml = sm_o + kConsumerWarps * 16 * kDh;               // [4][16][2]
  {
    float* ow = sm_o + warp * 16 * kDh;
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) {
      ow[g * kDh + nt * 8 + 2 * t] = o[nt][0];
      ow[g * kDh + nt * 8 + 2 * t + 1] = o[nt][1];
      ow[(g + 8) * kDh + nt * 8 + 2 * t] = o[nt][2];
      ow[(g + 8) * kDh + nt * 8 + 2 * t + 1] = o[nt][3];
    }
    if (t == 0) {
      sm_ml[(warp * 16 + g) * 2 + 0] = m0;
      sm_ml[(warp * 16 + g) * 2 + 1] = l0;
      sm_ml[(warp * 16 + g + 8) * 2 + 0] = m1;
      sm_ml[(warp * 16 + g + 8) * 2 + 1] = l1;
    }
  }
  named_barrier_sync(1, kConsumerWarps * 32);
  const int tid = threadIdx.x;  // 0..127 : one head dim each
  const bool split = it.n_splits > 1;
  for (int r = 0; r < G; ++r) {
    float mm = -INFINITY;
    for (int w = 0; w < kConsumerWarps; ++w) mm = fmaxf(mm, sm_ml[(w * 16 + r) * 2]);
    float base = mm == -INFINITY ? 0.f : mm;
    float ll = 0.f, acc = 0.f;
    for (int w = 0; w < kConsumerWarps; ++w) {
      float f = exp2f(sm_ml[(w * 16 + r) * 2] - base);
      ll += sm_ml[(w * 16 + r) * 2 + 1] * f;
      acc += sm_o[(w * 16 + r) * kDh + tid] * f;
    }
    if (!split) {
      bf16* dst = p.out + ((size_t)(q_base) * p.n_q_heads + kvh * G + r) * kDh;
      dst[tid] = f2bf(acc / ll);
    } else {
      // partial (unnormalised) result for this split
      size_t wi = ((size_t)it.ws_index * p.n_kv_heads + kvh) * G + r;
      p.ws_o[wi * kDh + tid] = acc;
      if (tid == 0) {
        p.ws_ml[wi * 2 + 0] = mm;
        p.ws_ml[wi * 2 + 1] = ll;
      }
    }
  }
  if (!split) return;
  // last CTA of this (seq, kv head) merges the splits
  __threadfence();
  named_barrier_sync(1, kConsumerWarps * 32);
  if (tid == 0) {
    int* ctr = p.counters + (size_t)it.seq * p.n_kv_heads + kvh;
    int prev = atomicAdd(ctr, 1);
    int last = prev == it.n_splits - 1;
    if (last) *ctr = 0;  // self-reset for the next launch
    *flag = last;
  }
  named_barrier_sync(1, kConsumerWarps * 32);
  if (!*flag) return;
  __threadfence();
  const int ws0 = it.ws_index - it.split;  // first split's workspace slot
  for (int r = 0; r < G; ++r) {
    float mm = -INFINITY;
    for (int sp = 0; sp < it.n_splits; ++sp) {
      size_t wi = ((size_t)(ws0 + sp) * p.n_kv_heads + kvh) * G + r;
      mm = fmaxf(mm, __ldcg(&p.ws_ml[wi * 2]));
    }
    float base = mm == -INFINITY ? 0.f : mm;
    float ll = 0.f, acc = 0.f;
    for (int sp = 0; sp < it.n_splits; ++sp) {
      size_t wi = ((size_t)(ws0 + sp) * p.n_kv_heads + kvh) * G + r;
      float f = exp2f(__ldcg(&p.ws_ml[wi * 2]) - base);
      ll += __ldcg(&p.ws_ml[wi * 2 + 1]) * f;
      acc += __ldcg(&p.ws_o[wi * kDh + tid]) * f;
    }
    bf16* dst = p.out + ((size_t)(q_base) * p.n_q_heads + kvh * G + r) * kDh;
    dst[tid] = f2bf(acc / ll);
  }
}

// ===========================================================================
// K1 persistent decode attention with a balanced schedule.
//
// The host cuts the decode work (every (sequence, kv head) pair's 64-key
// stages) into one contiguous range of equal length per CTA (stream-K style);
// a range may start or end inside a sequence, which then has several key
// segments merged through the split workspace by the last one to finish. The
// producer warp streams the paged K/V of all of a CTA's segments back to back
// (TMA, 3-stage ring), so the memory pipe never drains between sequences; the
// 4 consumer warps take interleaved 16-key blocks and merge per segment in a
// small dedicated shared buffer.
// ===========================================================================
namespace {
constexpr int kDecMaxG = 5;  // Llama-3 (4) and Qwen2.5 (5) groups; larger groups use paged_attention_kernel
constexpr int kDecSmem = 1024 + kStages * kStageBytes + kConsumerWarps * kDecMaxG * (kDh + 2) * 4 + 256;
}  // namespace

// One decode instance = 5 warps (warp 4 = TMA producer, warps 0-3 consumers)
// over the segments of virtual CTA `vcta`, on `smem` (kDecSmemInst bytes,
// 1024-aligned). bar_init (160 threads) / bar_cons (128 consumer threads) are
// the instance's named barriers.
// the instance's mbarriers: full[kStages] then empty[kStages]
PPD_DEV uint64_t* decode_bars(uint8_t* smem) {
  return reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes +
                                     (kConsumerWarps * kDecMaxG * kDh + kConsumerWarps * kDecMaxG * 2) * 4);
}

PPD_DEV void decode_body(const CUtensorMap* kv_map, const AttnParams& p, uint8_t* smem, int vcta, int warp, int lane,
                         int bar_init, int bar_cons) {
  uint8_t* stage_base = smem;
  float* mo = reinterpret_cast<float*>(smem + kStages * kStageBytes);  // [warp][G][Dh]
  float* mml = mo + kConsumerWarps * kDecMaxG * kDh;                    // [warp][G][2]
  uint64_t* full_bar = decode_bars(smem);
  uint64_t* empty_bar = full_bar + kStages;
  int* flag = reinterpret_cast<int*>(empty_bar + kStages);

  const int G = p.group;
  const int seg0 = p.seg_start[vcta], seg1 = p.seg_start[vcta + 1];

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], kConsumerWarps);
    }
    fence_barrier_init();
  }
  named_barrier_sync(bar_init, kThreads);

  if (warp == kConsumerWarps) {
    // the 16 boxes of a stage (4 blocks x K|V x two 64-dim halves): one lane each
    const int b = lane >> 2, is_v = (lane >> 1) & 1, h = lane & 1;
    // overlap: cached K/V (positions < ctx) was written by earlier steps, so it
    // streams before the predecessor (RoPE + KV write of this step's rows)
    // retires; the first stage holding a position >= ctx waits for it
    const uint64_t kv_pol = l2_evict_first_policy();
    bool waited = !p.overlap;
    int g = 0;  // global stage counter across this CTA's segments
    for (int sg = seg0; sg < seg1; ++sg) {
      const AttnItem it = p.items[sg];
      const int kvh = it.pad[0];
      const int* btab = p.block_tables + (size_t)it.seq * p.max_blocks;
      const int first_blk = it.key_begin / kBT, last_blk = (it.key_end - 1) / kBT;
      const int nst = (last_blk - first_blk) / kStageBlocks + 1;
      const int new_pos = p.ctx[it.seq];
      for (int st = 0; st < nst; ++st, ++g) {
        const int slot = g % kStages;
        if (g >= kStages) mbar_wait(&empty_bar[slot], ((g / kStages) - 1) & 1);
        const int b0 = first_blk + st * kStageBlocks;
        const int nb = min(kStageBlocks, last_blk - b0 + 1);
        if (!waited && (b0 + nb) * kBT > new_pos) {
          pdl_wait();
          waited = true;
        }
        if (lane == 0) mbar_arrive_expect_tx(&full_bar[slot], nb * 2 * kBlockBytes);
        __syncwarp();
        if (lane < 16 && b < nb) {
          const int blk = btab[b0 + b];
          const int row = (((blk * p.n_layers + p.layer) * 2 + is_v) * p.n_kv_heads + kvh) * kBT;
          void* dst = stage_base + slot * kStageBytes + (b * 2 + is_v) * kBlockBytes + h * 2048;
          if (p.l2_hint)  // cached K/V is read once per step
            tma_load_2d_hint(dst, kv_map, h * 64, row, &full_bar[slot], kv_pol);
          else
            tma_load_2d(dst, kv_map, h * 64, row, &full_bar[slot]);
        }
      }
    }
    pdl_trigger();
    return;
  }

  // ---------------- consumer warps ----------------
  if (p.overlap) {  // q is written by the predecessor
    pdl_wait();
    pdl_trigger();
  }
  const int g8 = lane >> 2, t = lane & 3;
  const float sl2 = p.scale_log2;
  const int tid = warp * 32 + lane;  // 0..127
  int g = 0;
  for (int sg = seg0; sg < seg1; ++sg) {
    const AttnItem it = p.items[sg];
    const int kvh = it.pad[0];
    const int s = it.seq;
    const int pos = p.ctx[s];
    const int q_base = p.q_start[s];
    const int key_begin = it.key_begin, key_end = it.key_end;
    const int first_blk = key_begin / kBT, last_blk = (key_end - 1) / kBT;
    const int nst = (last_blk - first_blk) / kStageBlocks + 1;
    // Q fragments: rows 0..G-1 are the G heads of this kv head (rows >= G zero)
    uint32_t qa[8][4];
    {
      const uint32_t* q0 = g8 < G ? reinterpret_cast<const uint32_t*>(p.q + ((size_t)q_base * p.n_q_heads + kvh * G + g8) * kDh)
                                  : nullptr;
      const uint32_t* q1 = (g8 + 8) < G ? reinterpret_cast<const uint32_t*>(
                                              p.q + ((size_t)q_base * p.n_q_heads + kvh * G + g8 + 8) * kDh)
                                        : nullptr;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int w0 = (kk * 16 + 2 * t) >> 1;
        qa[kk][0] = q0 ? __ldg(q0 + w0) : 0u;
        qa[kk][1] = q1 ? __ldg(q1 + w0) : 0u;
        qa[kk][2] = q0 ? __ldg(q0 + w0 + 4) : 0u;
        qa[kk][3] = q1 ? __ldg(q1 + w0 + 4) : 0u;
      }
    }
    float o[16][4];
#pragma unroll
    for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    for (int st = 0; st < nst; ++st, ++g) {
      const int slot = g % kStages;
      mbar_wait(&full_bar[slot], (g / kStages) & 1);
      const int stage_blocks_valid = min(kStageBlocks, last_blk - (first_blk + st * kStageBlocks) + 1);
      if (warp < stage_blocks_valid) {
        const uint32_t kb = smem_u32(stage_base + slot * kStageBytes) + (warp * 2 + 0) * kBlockBytes;
        const uint32_t vb = kb + kBlockBytes;
        float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4(kb + kv_off((lane & 7) + (lane >> 4) * 8, kk * 16 + ((lane >> 3) & 1) * 8), b0, b1, b2, b3);
          mma16816(sc[0], qa[kk], b0, b1);
          mma16816(sc[1], qa[kk], b2, b3);
        }
        const int key = (first_blk + st * kStageBlocks + warp) * kBT;
        float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int k = key + nt * 8 + 2 * t + e;
            const bool ok = k >= key_begin && k < key_end && k <= pos;
            sc[nt][e] = ok ? sc[nt][e] * sl2 : -INFINITY;
            sc[nt][2 + e] = ok ? sc[nt][2 + e] * sl2 : -INFINITY;
            mx0 = fmaxf(mx0, sc[nt][e]);
            mx1 = fmaxf(mx1, sc[nt][2 + e]);
          }
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
        const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
        const float base0 = mn0 == -INFINITY ? 0.f : mn0, base1 = mn1 == -INFINITY ? 0.f : mn1;
        const float corr0 = exp2f(m0 - base0), corr1 = exp2f(m1 - base1);
        m0 = mn0;
        m1 = mn1;
        const float p00 = exp2f(sc[0][0] - base0), p01 = exp2f(sc[0][1] - base0);
        const float p02 = exp2f(sc[0][2] - base1), p03 = exp2f(sc[0][3] - base1);
        const float p10 = exp2f(sc[1][0] - base0), p11 = exp2f(sc[1][1] - base0);
        const float p12 = exp2f(sc[1][2] - base1), p13 = exp2f(sc[1][3] - base1);
        float rs0 = p00 + p01 + p10 + p11, rs1 = p02 + p03 + p12 + p13;
        rs0 += __shfl_xor_sync(0xffffffffu, rs0, 1);
        rs0 += __shfl_xor_sync(0xffffffffu, rs0, 2);
        rs1 += __shfl_xor_sync(0xffffffffu, rs1, 1);
        rs1 += __shfl_xor_sync(0xffffffffu, rs1, 2);
        l0 = l0 * corr0 + rs0;
        l1 = l1 * corr1 + rs1;
        const uint32_t a[4] = {pack2(p00, p01), pack2(p02, p03), pack2(p10, p11), pack2(p12, p13)};
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          o[i][0] *= corr0;
          o[i][1] *= corr0;
          o[i][2] *= corr1;
          o[i][3] *= corr1;
        }
#pragma unroll
        for (int nt = 0; nt < 16; nt += 2) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(vb + kv_off((lane & 7) + ((lane >> 3) & 1) * 8, nt * 8 + (lane >> 4) * 8), b0, b1, b2, b3);
          mma16816(o[nt], a, b0, b1);
          mma16816(o[nt + 1], a, b2, b3);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[slot]);
    }
    // ---- merge the 4 warps (rows < G) through the dedicated buffer
    if (g8 < G) {
      float* ow = mo + (warp * kDecMaxG + g8) * kDh;
#pragma unroll
      for (int nt = 0; nt < 16; ++nt) sts_f32x2(ow + nt * 8 + 2 * t, o[nt][0], o[nt][1]);
      if (t == 0) sts_f32x2(mml + (warp * kDecMaxG + g8) * 2, m0, l0);
    }
    named_barrier_sync(bar_cons, kConsumerWarps * 32);
    const bool split = it.n_splits > 1;
    for (int r = 0; r < G; ++r) {
      float mm = -INFINITY;
      for (int w = 0; w < kConsumerWarps; ++w) mm = fmaxf(mm, lds_f32(mml + (w * kDecMaxG + r) * 2));
      const float base = mm == -INFINITY ? 0.f : mm;
      float ll = 0.f, acc = 0.f;
      for (int w = 0; w < kConsumerWarps; ++w) {
        const float f = exp2f(lds_f32(mml + (w * kDecMaxG + r) * 2) - base);
        ll += lds_f32(mml + (w * kDecMaxG + r) * 2 + 1) * f;
        acc += lds_f32(mo + (w * kDecMaxG + r) * kDh + tid) * f;
      }
      if (!split) {
        p.out[((size_t)q_base * p.n_q_heads + kvh * G + r) * kDh + tid] = f2bf(acc / ll);
      } else {
        const size_t wi = ((size_t)it.ws_index * p.n_kv_heads + kvh) * G + r;
        p.ws_o[wi * kDh + tid] = acc;
        if (tid == 0) {
          p.ws_ml[wi * 2 + 0] = mm;
          p.ws_ml[wi * 2 + 1] = ll;
        }
      }
    }
    if (split) {
      // release / acquire through one thread (the cooperative-groups grid
      // barrier pattern): the CTA barrier orders every consumer's workspace
      // stores before thread 0's fence + counter update, and the last
      // arriver's fence before the barrier that releases its merge reads
      named_barrier_sync(bar_cons, kConsumerWarps * 32);
      if (tid == 0) {
        int* ctr = p.counters + (size_t)s * p.n_kv_heads + kvh;
        __threadfence();
        const int prev = atomicAdd(ctr, 1);
        const int last = prev == it.n_splits - 1;
        if (last) {
          *ctr = 0;
          __threadfence();
        }
        *flag = last;
      }
      named_barrier_sync(bar_cons, kConsumerWarps * 32);
      if (*flag) {
        const int ws0 = it.ws_index - it.split;
        const int ns = it.n_splits;
        // the host cuts at most 2 * 148 ranges: ns * G (m, l) pairs fit the
        // merge buffer for every kv-head count >= 2 at G <= kDecMaxG
        if (2 * ns * G > kConsumerWarps * kDecMaxG * kDh) __trap();
        // every split's (m, l) of every row staged in the (consumed) merge
        // buffer by one load per thread, then all rows' partial outputs of 4
        // splits at a time in flight: these were serial L2 round trips per
        // row and split (~10 us on the last CTA of a split sequence). Same
        // summation order (split ascending) as a row-by-row merge.
        for (int i = tid; i < ns * G; i += kConsumerWarps * 32) {
          const int sp = i / G, r = i - sp * G;
          const size_t wi = ((size_t)(ws0 + sp) * p.n_kv_heads + kvh) * G + r;
          const float2 ml = __ldcg(reinterpret_cast<const float2*>(p.ws_ml) + wi);
          sts_f32x2(mo + 2 * i, ml.x, ml.y);
        }
        named_barrier_sync(bar_cons, kConsumerWarps * 32);
        float base[kDecMaxG], ll[kDecMaxG], acc[kDecMaxG];
#pragma unroll
        for (int r = 0; r < kDecMaxG; ++r) {
          float mm = -INFINITY;
          if (r < G)
            for (int sp = 0; sp < ns; ++sp) mm = fmaxf(mm, lds_f32(mo + 2 * (sp * G + r)));
          base[r] = mm == -INFINITY ? 0.f : mm;
          ll[r] = 0.f;
          acc[r] = 0.f;
        }
        for (int sp0 = 0; sp0 < ns; sp0 += 4) {
          float v[kDecMaxG][4];
#pragma unroll
          for (int r = 0; r < kDecMaxG; ++r)
#pragma unroll
            for (int j = 0; j < 4; ++j)
              v[r][j] = (r < G && sp0 + j < ns)
                            ? __ldcg(&p.ws_o[(((size_t)(ws0 + sp0 + j) * p.n_kv_heads + kvh) * G + r) * kDh + tid])
                            : 0.f;
#pragma unroll
          for (int r = 0; r < kDecMaxG; ++r)
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (r < G && sp0 + j < ns) {
                const float* ml = mo + 2 * ((sp0 + j) * G + r);
                const float f = exp2f(lds_f32(ml) - base[r]);
                ll[r] += lds_f32(ml + 1) * f;
                acc[r] += v[r][j] * f;
              }
        }
#pragma unroll
        for (int r = 0; r < kDecMaxG; ++r)
          if (r < G) p.out[((size_t)q_base * p.n_q_heads + kvh * G + r) * kDh + tid] = f2bf(acc[r] / ll[r]);
      }
    }
    named_barrier_sync(bar_cons, kConsumerWarps * 32);  // merge buffer / flag reused by the next segment
  }
  pdl_trigger();
}

__global__ void __launch_bounds__(kThreads, 2)
    decode_attention_kernel(const __grid_constant__ CUtensorMap kv_map, AttnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  if (!p.overlap) pdl_wait();
  decode_body(&kv_map, p, smem, blockIdx.x, threadIdx.x >> 5, threadIdx.x & 31, 0, 1);
}

// ===========================================================================
// K2: ONE launch for a mixed decode + (append-)prefill step.
//
// CTAs [0, n_pf) start on the prefill queue: the K3/K4 tcgen05 tile of
// attention_tc_body.cuh on all 12 warps (TMEM allocated on entering the mode,
// mbarriers re-armed per tile), tiles pulled longest first with an atomic.
// Every other CTA runs TWO decode instances (warps 0-4 and 5-9, own smem
// ring and named barriers) over its two virtual CTAs of the balanced decode
// schedule (static: the host cut it for 2 x (gridDim.x - n_pf) instances, so
// the memory pipe streams without queue round trips), then joins the prefill
// queue. HBM-bound decode streaming and tensor-core-bound prefill tiles run
// concurrently on disjoint SMs; what prefill work is left when decode ends is
// shared by every SM. Queue head + done counter live in p.mix_ctr[0..1]; the
// last CTA out resets them for the next launch.
// ===========================================================================
namespace {
constexpr int kMixSW = 8;  // softmax warps of the prefill role (2 threads per query row)
constexpr int kMixThreads = pftc::threads_for(kMixSW);  // 384: the prefill role's 12 warps (decode uses 10)
constexpr int kDecSmemInst = (kDecSmem - 1024 + 1023) / 1024 * 1024;
constexpr int kMixSmem = pftc::kSmem > 1024 + 2 * kDecSmemInst ? pftc::kSmem : 1024 + 2 * kDecSmemInst;
constexpr int kMixBarAll = 1;   // all 320 threads: mode switch
constexpr int kMixBarPf = 2;    // prefill warps 0-7
constexpr int kMixBarDec = 3;   // decode instance i: 3 + i (160 threads), consumers 5 + i (128)
}  // namespace

__global__ void __launch_bounds__(kMixThreads, 1)
    mixed_attention_kernel(const __grid_constant__ CUtensorMap kv_map, AttnParams p, const AttnItem* pf_items,
                           int n_pf, int n_pf_tiles, int n_vcta) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ int s_next;
  pdl_wait();
  if (p.overlap) pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if ((int)blockIdx.x >= n_pf) {
    // ---------------- decode: two static virtual CTAs, then help with prefill
    const int inst = threadIdx.x / kThreads;
    const int lt = threadIdx.x - inst * kThreads;
    const int v = ((int)blockIdx.x - n_pf) * 2 + inst;
    if (inst < 2 && v < n_vcta)
      decode_body(&kv_map, p, smem + inst * kDecSmemInst, v, lt >> 5, lt & 31, kMixBarDec + inst,
                  kMixBarDec + 2 + inst);
    named_barrier_sync(kMixBarAll, kMixThreads);  // both instances retired: smem free
    // the prefill role reuses this smem for tiles and its own barriers: the
    // decode instances' mbarrier objects are invalidated first (PTX: a
    // location holding an mbarrier is repurposed only after mbarrier.inval)
    if (threadIdx.x < 2 && ((int)blockIdx.x - n_pf) * 2 + (int)threadIdx.x < n_vcta) {
      uint64_t* bars = decode_bars(smem + threadIdx.x * kDecSmemInst);
      for (int i = 0; i < 2 * kStages; ++i)
        asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(bars + i)) : "memory");
    }
    named_barrier_sync(kMixBarAll, kMixThreads);
  }
  // ---------------- prefill queue (all 12 warps)
  pftc::tile_queue<kMixSW>(&kv_map, p, smem, pf_items, n_pf_tiles, warp, lane, kMixBarPf, p.mix_ctr, p.mix_ctr + 1,
                     gridDim.x, &s_next);
  pdl_trigger();
}

cudaError_t launch_mixed_attention(const void* kv_map, const AttnParams& p, const AttnItem* pf_items, int n_pf,
                                   int n_pf_tiles, int n_vcta, cudaStream_t stream) {
  static unsigned long long attr_devs = 0;
  if (first_on_device(&attr_devs)) {
    cudaFuncSetAttribute(mixed_attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMixSmem);
  }
  if (p.group > kDecMaxG || n_pf <= 0 || n_pf > n_pf_tiles || !p.mix_ctr) return cudaErrorInvalidValue;
  const int grid = n_pf + (n_vcta + 1) / 2;
  return launch_pdl(mixed_attention_kernel, dim3(grid), dim3(kMixThreads), kMixSmem, stream,
                    *reinterpret_cast<const CUtensorMap*>(kv_map), p, pf_items, n_pf, n_pf_tiles, n_vcta);
}

cudaError_t launch_decode_attention(const void* kv_map, const AttnParams& p, int n_cta, int group,
                                    cudaStream_t stream) {
  static unsigned long long attr_devs = 0;
  if (first_on_device(&attr_devs)) {
    cudaFuncSetAttribute(decode_attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kDecSmem);
  }
  if (n_cta == 0) return cudaSuccess;
  if (group > kDecMaxG) return cudaErrorInvalidValue;
  return launch_pdl(decode_attention_kernel, dim3(n_cta), dim3(kThreads), kDecSmem, stream,
                    *reinterpret_cast<const CUtensorMap*>(kv_map), p);
}

// ---------------------------------------------------------------------------

static PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* ptr = nullptr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q);
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

int make_kv_tensor_map(void* map_out, const void* pool, uint64_t total_rows) {
  auto fn = get_encode_fn();
  if (!fn) return -1;
  cuuint64_t dims[2] = {(cuuint64_t)kDh, (cuuint64_t)total_rows};
  cuuint64_t strides[1] = {(cuuint64_t)kDh * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)kBT};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(reinterpret_cast<CUtensorMap*>(map_out), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                  const_cast<void*>(pool), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -(int)r;
}

cudaError_t launch_paged_attention(const void* kv_map, const AttnParams& p, int n_items,
                                   cudaStream_t stream) {
  static unsigned long long attr_devs = 0;
  if (first_on_device(&attr_devs)) {
    cudaFuncSetAttribute(paged_attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
  }
  if (n_items == 0) return cudaSuccess;
  dim3 grid(n_items, p.n_kv_heads);
  return launch_pdl(paged_attention_kernel, grid, dim3(kThreads), kSmemBytes, stream,
                    *reinterpret_cast<const CUtensorMap*>(kv_map), p);
}

}  // namespace ppdk
