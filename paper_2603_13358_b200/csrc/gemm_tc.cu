// gemm_tc.cu — K5: hand-written tcgen05/TMEM/TMA GEMM for the projection, MLP
// and lm_head contractions:  C[T][N] = X[T][K] . W[N][K]^T  (bf16 in, fp32 acc).
//
// Weight rows are the UMMA M dimension (128 per CTA tile) and tokens the UMMA N
// dimension (BN <= 256 per tile), so a decode batch of B <= 256 tokens is ONE
// token tile and every CTA streams a disjoint 128-row slab of the weights
// (the decode step is weight-streaming, HBM-bound); prefill (thousands of
// tokens) tiles the token dimension too and becomes tensor-core bound. When
// the (weight tile x token tile) grid cannot fill the 148 SMs the K loop is
// split and each split writes an fp32 partial slice; the consumer kernel
// (RMSNorm / RoPE) sums the slices, so no extra reduction launch exists.
//
// Warp roles (256 threads): warp 0 = TMA producer (one elected lane), warp 1 =
// MMA issuer (one lane, tcgen05.mma.cta_group::1.kind::f16, accumulator in
// TMEM), warp 2 = TMEM allocator, warps 4-7 = epilogue (tcgen05.ld 32x32b,
// each warp owns TMEM lanes 32*(w%4)...). smem operands are TMA-loaded with
// the 128-byte swizzle and described to the tensor core by SW128 K-major
// UMMA descriptors; a 4..8-stage mbarrier ring keeps TMA ahead of the MMAs.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "gemm_tc.h"
#include "kernels.h"

namespace ppdk {

namespace {

constexpr int kBK = 64;                       // K elements per stage (128 B rows)
constexpr int kBM = 128;                      // weight rows per tile (UMMA M)
constexpr int kMaxBN = 256;                   // tokens per tile (UMMA N)
constexpr int kThreads = 256;
constexpr int kWBytes = kBM * kBK * 2;        // 16 KB
constexpr int kSmemBudget = 220 * 1024;
constexpr int kMaxStages = 8;
constexpr int kBarBytes = 256;                // mbarriers + TMEM slot after the stage ring
constexpr int kXchgBytes = 2 * 2 * 32 * 32 * 4;  // fused epilogue: 2 buffers x 2 warps x 32x32 fp32
constexpr int kEpiPlain = 0, kEpiSilu = 1;

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

// prefetch one box of a tensor-mapped matrix into L2 (no smem, no completion)
PPD_DEV void tma_prefetch_l2(const CUtensorMap* map, int x, int y) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y)
               : "memory");
}

PPD_DEV uint64_t sw128_kmajor_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);   // start address
  d |= (uint64_t)1 << 16;                    // LBO (unused for swizzled K-major) = 16 B
  d |= (uint64_t)(1024 >> 4) << 32;          // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                    // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                    // SWIZZLE_128B
  return d;
}

PPD_DEV void mma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

PPD_DEV void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

PPD_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
PPD_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

PPD_DEV void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// the same load without the wait: the registers are valid only after wait_tmem_ld()
PPD_DEV void tmem_ld32_async(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}
PPD_DEV void wait_tmem_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// store 32 token columns of one output row (fp32 or bf16), token stride ldo;
// one running pointer (32 precomputed 64-bit addresses cost 64 registers)
template <bool kF32>
PPD_DEV void store_cols32(void* base, size_t ldo, const uint32_t* r, int nj) {
  if (kF32) {
    float* d = static_cast<float*>(base);
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) {
      if (jj < nj) *d = __uint_as_float(r[jj]);
      d += ldo;
    }
  } else {
    __nv_bfloat16* d = static_cast<__nv_bfloat16*>(base);
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) {
      if (jj < nj) *d = __float2bfloat16_rn(__uint_as_float(r[jj]));
      d += ldo;
    }
  }
}

// ---- CTA-pair (cta_group::2) primitives ------------------------------------
PPD_DEV uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cta address in this CTA -> shared::cluster address of the same offset in CTA `rank`
PPD_DEV uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
PPD_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA into this CTA's smem, completion bytes counted on the leader CTA's mbarrier
PPD_DEV void tma_load_2d_pair(void* smem, const CUtensorMap* map, int x, int y, uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar_cluster)
      : "memory");
}
PPD_DEV void tma_load_2d_pair_hint(void* smem, const CUtensorMap* map, int x, int y, uint32_t bar_cluster,
                                   uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar_cluster), "l"(pol)
      : "memory");
}
PPD_DEV void mma_bf16_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}
// arrive (once the issued MMAs retire) on the barrier at this offset in both CTAs of the pair
PPD_DEV void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
PPD_DEV void mbar_arrive_remote(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}
PPD_DEV void mbar_wait_cluster(uint64_t* bar, uint32_t phase) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n.reg .pred p;\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}

}  // namespace

// ---- work schedule shared by the producer, MMA and epilogue roles ----------
// A segment is a contiguous k-block range [kb0, kb1) of one (weight tile,
// token tile) whose accumulator goes to partial slice `slice`.
//  * uniform: units (tile, split) dealt round-robin to the slots;
//  * balanced: the first `dp` tiles (whole waves of whole-K units) are dealt
//    round-robin, so consecutive slots share a weight tile at the same
//    k-block (its weights come from HBM once, from L2 for the other token
//    tiles); the remaining (tile, k-block) items, `total` of them, are cut
//    into `tail_slots` equal contiguous ranges, slot c < tail_slots owning
//    [c*total/tail_slots, (c+1)*total/tail_slots) (stream-K tail: no wave
//    quantization). GemmParts documents the slice rule.
struct Seg {
  int tw, tt, kb0, kb1, slice;
};
struct Sched {
  int n_tiles_t, kbt, kb_per, splits, n_units, slots, c, u;
  int balanced, dp, tslots;
  long long total, x, end;

  PPD_DEV void begin(const GemmTcParams& p, int rows, int c_, int slots_) {
    n_tiles_t = (p.T + p.bn * p.n_sub - 1) / (p.bn * p.n_sub);
    kbt = (p.K + kBK - 1) / kBK;
    splits = p.splits;
    kb_per = (kbt + splits - 1) / splits;
    n_units = ((p.N + rows - 1) / rows) * n_tiles_t * splits;
    slots = slots_;
    c = c_;
    u = c_;
    balanced = p.balanced;
    dp = p.dp;
    tslots = p.tail_slots;
    total = p.total;
    x = end = 0;
    if (balanced && c_ < tslots) {
      x = (long long)c_ * total / tslots;
      end = (long long)(c_ + 1) * total / tslots;
    }
  }
  PPD_DEV int owner(long long item) const { return (int)(((item + 1) * tslots + total - 1) / total) - 1; }
  PPD_DEV bool next(Seg& s) {
    if (!balanced) {
      if (u >= n_units) return false;
      s.slice = u % splits;
      const int rest = u / splits;
      s.tt = rest % n_tiles_t;
      s.tw = rest / n_tiles_t;
      s.kb0 = s.slice * kb_per;
      s.kb1 = min(kbt, s.kb0 + kb_per);
      u += slots;
      return true;
    }
    if (u < dp) {  // data-parallel waves: whole K, slice 0
      s.tt = u % n_tiles_t;
      s.tw = u / n_tiles_t;
      s.kb0 = 0;
      s.kb1 = kbt;
      s.slice = 0;
      u += slots;
      return true;
    }
    if (x >= end) return false;
    const long long t = x / kbt;
    s.kb0 = (int)(x - t * kbt);
    s.kb1 = (int)min((long long)kbt, s.kb0 + (end - x));
    s.tt = (int)((t + dp) % n_tiles_t);
    s.tw = (int)((t + dp) / n_tiles_t);
    s.slice = c - owner(t * kbt);
    x += s.kb1 - s.kb0;
    return true;
  }
};

// Persistent GEMM. kPair = false: one CTA per slot, 128-row weight tiles,
// tcgen05 cta_group::1. kPair = true: a cluster of 2 CTAs on one TPC per slot,
// 256-row weight tiles, UMMA M=256 with cta_group::2: CTA r streams weight rows
// [128r, 128r+128) of the tile and HALF of the token tile (bn/2 rows), and
// the leader's single-thread MMA reads both CTAs' shared memory.
//
// One TMA ring of stages (16 KB of weights + the k-block's activation tile,
// one mbarrier transaction). Weights do not depend on the previous kernel:
// the producer streams the first ring's worth of weight tiles before
// griddepcontrol.wait (PDL), then the activations. (Measured: splitting the
// activations into their own shallow ring with a second producer warp is
// 20-30% slower at T=200 — tools/ab_libs.py.)
//
// The MMA warp alternates between two TMEM accumulators (when 2*BN <= 512
// columns) so the epilogue of segment i overlaps the MMAs of segment i+1.
// Pair protocol: both CTAs' TMAs complete on the LEADER's full barrier (the
// leader alone arms it with both CTAs' bytes); the leader's commits multicast
// to the smem-slot and accumulator barriers of both CTAs; both epilogues
// release an accumulator on the leader's barrier (8 warp arrivals).
template <bool kPair, int kEpi, int kOcc, int kNSub>
__global__ void __launch_bounds__(kThreads, kOcc)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x,
                   GemmTcParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int kCta = kPair ? 2 : 1;
  const int S = p.stages;
  const int xrows = p.bn / kCta;  // token rows this CTA loads per stage and token sub-tile
  // kNSub token sub-tiles of bn rows per unit (compile time): one weight stage feeds kNSub MMAs
  const int unit_t = p.bn * kNSub;
  const int stage_bytes = kWBytes + kNSub * xrows * kBK * 2;  // multiples of 1 KB
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);
  uint64_t* empty = full + S;
  uint64_t* acc_full = empty + S;      // [2]
  uint64_t* acc_empty = acc_full + 2;  // [2] (pair: used in the leader only)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  float* xchg = reinterpret_cast<float*>(smem + S * stage_bytes + kBarBytes);  // fused-epilogue exchange

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = kPair ? cluster_ctarank() : 0;
  const bool leader = rank == 0;
  const int slot = kPair ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int n_slots = kPair ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int acc_cols = kNSub * p.bn_cols;  // TMEM columns of one accumulator set
  const int n_acc = p.tmem_cols >= 2 * acc_cols ? 2 : 1;

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 4 * kCta);  // one arrive per epilogue warp (of both CTAs)
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    if (kPair) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(p.tmem_cols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(p.tmem_cols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (kPair) cluster_sync_all();  // peer barriers initialised + TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // the next kernel may launch; it waits for our completion itself. overlap:
  // only once our own predecessor retired (pdl_enter in common.cuh)
  if (!p.overlap) pdl_trigger();

  const int rows = kBM * kCta;
  const uint32_t full_bar0 = kPair ? mapa_shared(smem_u32(full), 0) : smem_u32(full);
  const uint32_t acc_empty0 = kPair ? mapa_shared(smem_u32(acc_empty), 0) : smem_u32(acc_empty);
  const int w_row0 = (int)rank * kBM;
  const int x_row0 = (int)rank * xrows;
  const uint32_t tx_bytes = (uint32_t)(kCta * stage_bytes);

  auto load = [&](void* dst, const CUtensorMap* map, int x, int y, int s) {
    if (kPair)
      tma_load_2d_pair(dst, map, x, y, full_bar0 + 8u * s);
    else
      tma_load_2d(dst, map, x, y, &full[s]);
  };
  // weights are read once per step: evict-first in L2 (p.l2_hint)
  const uint64_t wpol = l2_evict_first_policy();
  auto load_w = [&](void* dst, int x, int y, int s) {
    if (!p.l2_hint)
      load(dst, &map_w, x, y, s);
    else if (kPair)
      tma_load_2d_pair_hint(dst, &map_w, x, y, full_bar0 + 8u * s, wpol);
    else
      tma_load_2d_hint(dst, &map_w, x, y, &full[s], wpol);
  };

  if (p.overlap && !(warp == 0 && lane == 0) && warp < 4) {  // every thread passes the wait before triggering
    pdl_wait();
    pdl_trigger();
  }
  if (warp == 0) {
    if (lane == 0) {
      Sched sc;
      sc.begin(p, rows, slot, n_slots);
      Seg sg;
      int npre = 0;
      {
        Sched pre = sc;
        while (npre < S && pre.next(sg)) {
          for (int kb = sg.kb0; kb < sg.kb1 && npre < S; ++kb, ++npre) {
            if (leader) mbar_arrive_expect_tx(&full[npre], tx_bytes);
            load_w(smem + npre * stage_bytes, kb * kBK, sg.tw * rows + w_row0, npre);
          }
        }
      }
      // and the next l2_pre k-blocks' weights into L2: the HBM pipe stays busy
      // through the predecessor's tail instead of idling until its outputs land
      if (p.l2_pre > 0) {
        Sched pre = sc;
        int idx = 0, done = 0;
        while (done < p.l2_pre && pre.next(sg)) {
          for (int kb = sg.kb0; kb < sg.kb1 && done < p.l2_pre; ++kb, ++idx) {
            if (idx < npre) continue;
            tma_prefetch_l2(&map_w, kb * kBK, sg.tw * rows + w_row0);
            ++done;
          }
        }
      }
      pdl_wait();
      if (p.overlap) pdl_trigger();
      int it = 0;  // global stage counter across segments
      while (sc.next(sg)) {
        for (int kb = sg.kb0; kb < sg.kb1; ++kb, ++it) {
          const int s = it % S;
          uint8_t* sw = smem + s * stage_bytes;
          if (it >= npre) {
            if (it >= S) {
              if (kPair)
                mbar_wait_cluster(&empty[s], ((it / S) - 1) & 1);
              else
                mbar_wait(&empty[s], ((it / S) - 1) & 1);
            }
            if (leader) mbar_arrive_expect_tx(&full[s], tx_bytes);
            load_w(sw, kb * kBK, sg.tw * rows + w_row0, s);
          }
#pragma unroll
          for (int jx = 0; jx < kNSub; ++jx)
            load(sw + kWBytes + jx * xrows * (kBK * 2), &map_x, kb * kBK, sg.tt * unit_t + jx * p.bn + x_row0, s);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(p.bn >> 3) << 17) |
                             ((uint32_t)(rows >> 4) << 24);
      Sched sc;
      sc.begin(p, rows, slot, n_slots);
      Seg sg;
      int it = 0, j = 0;
      for (; sc.next(sg); ++j) {
        const int acc = j % n_acc;
        const int use = j / n_acc;  // how many times this accumulator was used before
        if (use > 0) {
          if (kPair)
            mbar_wait_cluster(&acc_empty[acc], (use - 1) & 1);
          else
            mbar_wait(&acc_empty[acc], (use - 1) & 1);
        }
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * acc_cols);
        for (int kb = sg.kb0; kb < sg.kb1; ++kb, ++it) {
          const int s = it % S;
          mbar_wait(&full[s], (it / S) & 1);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + s * stage_bytes);
          const uint64_t da = sw128_kmajor_desc(sa);
#pragma unroll
          for (int js = 0; js < kNSub; ++js) {
            const uint64_t db = sw128_kmajor_desc(sa + kWBytes + js * xrows * (kBK * 2));
            const uint32_t dj = d_tmem + (uint32_t)(js * p.bn_cols);
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {  // 32 B per UMMA_K step inside the swizzle atom
              const uint32_t accum = (kb != sg.kb0) || (k != 0);
              if (kPair)
                mma_bf16_pair(dj, da + (uint64_t)(k * 2), db + (uint64_t)(k * 2), idesc, accum);
              else
                mma_bf16(dj, da + (uint64_t)(k * 2), db + (uint64_t)(k * 2), idesc, accum);
            }
          }
          if (kPair)
            mma_commit_pair(&empty[s]);  // smem slot (in both CTAs) free once these MMAs retire
          else
            mma_commit(&empty[s]);
        }
        if (kPair)
          mma_commit_pair(&acc_full[acc]);
        else
          mma_commit(&acc_full[acc]);
      }
    }
  } else if (warp >= 4) {
    pdl_wait();  // outputs are written only after the predecessor retired
    if (p.overlap) pdl_trigger();
    const int q = warp & 3;  // TMEM lane quarter owned by this warp
    Sched sc;
    sc.begin(p, rows, slot, n_slots);
    Seg sg;
    // SiLU exchange-buffer parity runs on across sub-tiles AND segments: warps
    // 2-3 may start the next segment's first chunk while warps 0-1 still read
    // the last chunk of this one (a per-segment reset raced there whenever a
    // segment ended on buffer 0; found by compute-sanitizer memcheck timing)
    int buf = 0;
    for (int j = 0; sc.next(sg); ++j) {
      const int acc = j % n_acc;
      const int use = j / n_acc;
      const int row = sg.tw * rows + w_row0 + q * 32 + lane;
      mbar_wait(&acc_full[acc], use & 1);
      tc_fence_after();
      float* out32 = reinterpret_cast<float*>(p.out) + (size_t)sg.slice * p.split_stride;
      __nv_bfloat16* out16 = reinterpret_cast<__nv_bfloat16*>(p.out);
#pragma unroll
      for (int jsub = 0; jsub < kNSub; ++jsub) {
      const int t0 = sg.tt * unit_t + jsub * p.bn;
      const uint32_t t_acc =
          tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * acc_cols + jsub * p.bn_cols);
      const int ncols = min(p.bn, p.T - t0);
      if (kEpi == kEpiSilu) {
        // Fused SiLU(gate) * up. The 128-row slab of this CTA is one interleaved
        // gate|up group (launch_fill_gate_up): TMEM lanes 0-63 = gate rows,
        // 64-127 = the matching up rows. Warps 2-3 hand their up values to
        // warps 0-1 through a double-buffered smem exchange; warps 0-1 write
        // m[t][64*group + lane'] = rbf(silu(g) * u) (same fp32 formula as
        // silu_mul_kernel, so the unfused path gives the same bits).
        const int grp = (sg.tw * rows + w_row0) / kBM;
        __nv_bfloat16* m = reinterpret_cast<__nv_bfloat16*>(p.out);
        for (int c0 = 0; c0 < ncols; c0 += 32, buf ^= 1) {
          uint32_t r[32];
          tmem_ld32(t_acc + (uint32_t)c0, r);
          float* xb = xchg + buf * 2048;
          if (q >= 2) {  // explicit st.shared (a generic store through xchg would be ST.E)
            const uint32_t xa = smem_u32(xb + (q - 2) * 1024 + lane);
#pragma unroll
            for (int jj = 0; jj < 32; ++jj)
              asm volatile("st.shared.b32 [%0], %1;" ::"r"(xa + 128u * jj), "r"(r[jj]) : "memory");
          }
          named_barrier_sync(1, 128);
          if (q < 2 && grp * kBM < p.N) {
            const int nj = min(32, ncols - c0);
            __nv_bfloat16* dst = m + (size_t)(t0 + c0) * p.ldo + grp * 64 + q * 32 + lane;
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) {
              if (jj < nj) {
                const float g = __uint_as_float(r[jj]);
                float u;
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(u) : "r"(smem_u32(xb + q * 1024 + jj * 32 + lane)) : "memory");
                dst[(size_t)jj * p.ldo] = __float2bfloat16_rn(__fmul_rn(__fdividef(g, __fadd_rn(1.0f, __expf(-g))), u));
              }
            }
          }
        }
      } else if (kOcc == 1 && p.epi_pipe) {
        // two register buffers: the TMEM load of chunk c+32 is in flight while
        // chunk c is stored (a load + wait per chunk serialised ~4 us of TMEM
        // latency per 100 KB epilogue, tools/tma_stream_probe.cu mode I)
        uint32_t ra[32], rb[32];
        const bool in = row < p.N;
        const size_t off = (size_t)t0 * p.ldo + row;
        void* base = p.out_f32 ? static_cast<void*>(out32 + off) : static_cast<void*>(out16 + off);
        const size_t step = (size_t)32 * p.ldo * (p.out_f32 ? 4 : 2);
        tmem_ld32_async(t_acc, ra);
        wait_tmem_ld();
        for (int c0 = 0; c0 < ncols; c0 += 64) {
          if (c0 + 32 < ncols) tmem_ld32_async(t_acc + (uint32_t)(c0 + 32), rb);
          if (in) {
            if (p.out_f32) store_cols32<true>(base, p.ldo, ra, ncols - c0);
            else store_cols32<false>(base, p.ldo, ra, ncols - c0);
          }
          base = static_cast<uint8_t*>(base) + step;
          wait_tmem_ld();
          if (c0 + 32 >= ncols) break;
          if (c0 + 64 < ncols) tmem_ld32_async(t_acc + (uint32_t)(c0 + 64), ra);
          if (in) {
            if (p.out_f32) store_cols32<true>(base, p.ldo, rb, ncols - c0 - 32);
            else store_cols32<false>(base, p.ldo, rb, ncols - c0 - 32);
          }
          base = static_cast<uint8_t*>(base) + step;
          wait_tmem_ld();
        }
      } else
      for (int c0 = 0; c0 < ncols; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(t_acc + (uint32_t)c0, r);
        if (row < p.N) {
          const size_t off = (size_t)(t0 + c0) * p.ldo + row;
          if (p.out_f32)
            store_cols32<true>(out32 + off, p.ldo, r, ncols - c0);
          else
            store_cols32<false>(out16 + off, p.ldo, r, ncols - c0);
        }
      }
      }  // token sub-tiles
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (kPair)
          mbar_arrive_remote(acc_empty0 + 8u * acc);
        else
          mbar_arrive(&acc_empty[acc]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (kPair) cluster_sync_all();  // the leader's MMAs may read the peer's smem until here
  if (warp == 2) {
    if (kPair)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(p.tmem_cols));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(p.tmem_cols));
  }
}

// ----------------------------------------------------------------- host side
namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* ptr = nullptr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q);
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

struct MapKey {
  const void* ptr;
  int rows, K, box_rows;
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && rows == o.rows && K == o.K && box_rows == o.box_rows;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    return std::hash<const void*>()(k.ptr) ^ (size_t(k.rows) * 1000003u) ^ (size_t(k.K) << 20) ^ size_t(k.box_rows);
  }
};

// K-major [rows][K] bf16 matrix, box = box_rows x 64 K-elements, 128 B swizzle
bool get_map(CUtensorMap* out, const void* ptr, int rows, int K, int box_rows) {
  static std::mutex mu;
  static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  MapKey key{ptr, rows, K, box_rows};
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return true;
  }
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUtensorMap m;
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, m);
  *out = m;
  return true;
}

}  // namespace

bool gemm_tc_map(void* map_out, const void* ptr, int rows, int K, int box_rows) {
  return get_map(static_cast<CUtensorMap*>(map_out), ptr, rows, K, box_rows);
}

// Tuning knobs (ppd_set_tuning): pair = -1 auto / 0 single-CTA / 1 CTA pair;
// stages = cap on the smem ring depth (0 = as many as fit); sched = -1 auto /
// 0 uniform K split / 1 balanced partition.
static int g_pair_mode = -1;
// T in (256, 512]: one unit covers both token sub-tiles. 1 auto (wide shapes +
// narrow ones whose pair tiles fill the SMs), 2 every shape (paired), 3 wide only
static int g_multi_sub = 1;
static int g_l2_hint = 3;  // bit 0: GEMM weights, bit 1: decode K/V loads evict-first in L2
static bool g_epi_pipe = true;   // plain epilogue: TMEM load of the next 32 columns in flight during the stores
static bool g_even_tiles = true;  // T > 256 in separate token tiles: equal tiles, not 256-row ones
void gemm_tc_set_even_tiles(bool on) { g_even_tiles = on; }
// two co-resident single CTAs per SM: -1 auto (<= kOcc2MaxT tokens; measured
// tools/gemm_knobs.py: +10-20% weight streaming at T = 64 / 128, neutral at
// T = 200, a loss with CTA pairs), 0 off, 1 whenever the shape allows
// Round 2 (r02l, after the L2 evict-first weight policy): the single CTA per
// SM with the full ring is faster at every measured size (tools/ab_step.py,
// profiles/ab_small_r02l.log: B=16 -1.5%, B=64 -2.2%, B=128 -5.5%, B=32 +0.3%),
// so auto is off by default; -1 restores the <= kOcc2MaxT rule
static int g_occ2 = 0;
constexpr int kOcc2MaxT = 128;
constexpr int kOcc2Smem = 113 * 1024;
static int g_stage_cap = 0;
static int g_sched = -1;
static int g_l2_pre = 0;  // measured: neutral to 1.5% slower at 8-32 k-blocks (tools/ab_step.py)
constexpr int kL2PreAuto = 16;  // weight k-blocks (16 KB each per CTA) prefetched into L2 ahead of the ring
void gemm_tc_set_l2_pre(int n) { g_l2_pre = n; }



// Auto policy for the CTA-pair kernel (measured, tools/gemm_tprobe.py): pairs
// pay off only when the activation ingress matters (>= 48 token rows) AND each
// slot streams several tiles (the pair's cluster launch/sync costs dominate
// one-tile-per-CTA GEMMs such as QKV / o-proj / down-proj of a decode step).
constexpr int kPairMinT = 48;
constexpr double kPairMinTilesPerSm = 1.4;

void gemm_tc_set_multi_sub(int mode) { g_multi_sub = mode; }
void gemm_tc_set_epi_pipe(bool on) { g_epi_pipe = on; }
void gemm_tc_set_l2_hint(int mask) { g_l2_hint = mask; }
int gemm_tc_l2_hint() { return g_l2_hint; }
void gemm_tc_set_occ2(int mode) { g_occ2 = mode; }

void gemm_tc_set_tuning(int pair_mode, int stage_cap, int sched) {
  g_pair_mode = pair_mode;
  g_stage_cap = stage_cap;
  g_sched = sched;
}

namespace {

struct Shape {
  bool pair;
  int bn, rows, stages, stage_bytes, smem, slots;  // slots = co-resident CTAs (single) or pairs
  int n_sub;   // token sub-tiles of bn rows per unit: a decode + append step of T <= 512 rows
               // streams each weight stage ONCE for all its tokens (2 MMAs of N = bn)
  int unit_t;  // token rows per unit = bn * n_sub
  int occ;     // co-resident CTAs per SM: 2 = half-depth ring and one <= 256-column
               // accumulator each, so one CTA's fill / epilogue tail overlaps the
               // other's weight streaming
};

// every kernel instantiation the launcher can pick
#define PPD_GEMM_KERNELS(X)                                                            \
  X(false, kEpiPlain, 1, 1) X(true, kEpiPlain, 1, 1) X(false, kEpiPlain, 1, 2)         \
  X(true, kEpiPlain, 1, 2) X(false, kEpiSilu, 1, 1) X(true, kEpiSilu, 1, 1)            \
  X(false, kEpiSilu, 1, 2) X(true, kEpiSilu, 1, 2) X(false, kEpiPlain, 2, 1) X(true, kEpiPlain, 2, 1)

using GemmKernel = void (*)(const CUtensorMap, const CUtensorMap, GemmTcParams);
GemmKernel pick_kernel(bool pair, int epi, int occ, int n_sub) {
#define PPD_PICK(P, E, O, N) \
  if (pair == P && epi == E && occ == O && n_sub == N) return gemm_tc_kernel<P, E, O, N>;
  PPD_GEMM_KERNELS(PPD_PICK)
#undef PPD_PICK
  return nullptr;
}

void set_smem_attrs() {
  static unsigned long long done_devs = 0;
  if (!first_on_device(&done_devs)) return;
  const int bytes = 1024 + kSmemBudget + kBarBytes;
#define PPD_ATTR(P, E, O, N)                                                                \
  cudaFuncSetAttribute(gemm_tc_kernel<P, E, O, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                       O == 2 ? kOcc2Smem : bytes);
  PPD_GEMM_KERNELS(PPD_ATTR)
#undef PPD_ATTR
}

int max_pair_slots(int smem, int occ) {
  static std::mutex mu;
  static std::unordered_map<int, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(smem * 4 + occ);
  if (it != cache.end()) return it->second;
  set_smem_attrs();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * 74 * occ);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, pick_kernel(true, kEpiPlain, occ, 1), &cfg) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    n = 0;
  }
  cache.emplace(smem * 4 + occ, n);
  return n;
}

// Auto mode for 257-512-row steps (two token sub-tiles per unit, one
// accumulator set): the CTA pair also when K is long (down projection:
// 41.7 vs 45.7 us at T=328), and never the balanced partition (uniform splits
// measured 4-30% faster per shape, 4% on the mixed step; tools/gemm_rot.py,
// tools/ab_step.py).
constexpr int kSubPairMinK = 8192;
Shape shape_for(int T, int N, int K, int extra_smem = 0, bool force_single = false) {
  Shape sh{};
  // two token sub-tiles per unit only where the weight-tile grid alone keeps
  // the SMs busy (gate|up) or the K loop is long enough to split (down); the
  // narrow projections (qkv, o) need the parallelism of separate token tiles
  // (tools/gemm_mixed.py: qkv at T=456 39 -> 26 us, o 30 -> 19 us)
  const bool wide = (N + kBM - 1) / kBM >= kPairMinTilesPerSm * device_sms() || K >= kSubPairMinK;
  // a narrow projection takes the paired two-sub-tile unit too when some
  // uniform K split of its 256-row pair tiles fills >= 90% of the pair slots in
  // ONE round (qkv, 24 pair tiles x 3: T=328 22.9 -> 20.2 us, T=456 25.2 ->
  // 23.3 us; o-proj, 16 x 4 = 64 of 74, stays on separate token tiles:
  // 16.4 -> 16.6 / 17.2 -> 19.5 us; tools/gemm_mixed.py)
  bool narrow_fill = false;
  {
    const int pt = (N + 2 * kBM - 1) / (2 * kBM), pslots = device_sms() / 2;
    for (int sp = 1; sp <= 8; ++sp)
      if (pt * sp <= pslots && pt * sp >= 0.9 * pslots) narrow_fill = true;
  }
  const bool narrow_pair = g_multi_sub == 2 || (g_multi_sub == 1 && narrow_fill && g_pair_mode != 0);
  if (T <= kMaxBN) {
    sh.n_sub = 1;
    sh.bn = ((T + 15) / 16) * 16;
  } else if (T <= 2 * kMaxBN && g_multi_sub && (wide || narrow_pair)) {
    sh.n_sub = 2;
    sh.bn = (((T + 1) / 2 + 15) / 16) * 16;
  } else {
    // equal token tiles (T=328: 2 x 176 rather than 256 + 72): shallower
    // activation stages, so a deeper ring
    const int ntt = (T + kMaxBN - 1) / kMaxBN;
    sh.n_sub = 1;
    sh.bn = g_even_tiles ? (((T + ntt - 1) / ntt + 15) / 16) * 16 : kMaxBN;
  }
  sh.unit_t = sh.bn * sh.n_sub;
  const double tiles1 = double((N + kBM - 1) / kBM) * ((T + sh.unit_t - 1) / sh.unit_t);
  // long-K (down projection) steps of > 1024 rows pair as well (T=2048: 232 -> 220 us)
  const bool auto_pair =
      T >= kPairMinT && (tiles1 >= kPairMinTilesPerSm * device_sms() || (sh.n_sub > 1 && K >= kSubPairMinK) ||
                         (sh.n_sub > 1 && narrow_pair) ||
                         (T > 4 * kMaxBN && K >= kSubPairMinK));
  const bool want_occ2 = sh.n_sub == 1 && extra_smem == 0 && (g_occ2 == 1 || (g_occ2 < 0 && T <= kOcc2MaxT));
  sh.pair = !force_single && (g_pair_mode == 1 || (g_pair_mode < 0 && auto_pair && !want_occ2));
  sh.rows = sh.pair ? 2 * kBM : kBM;
  sh.stage_bytes = kWBytes + sh.n_sub * (sh.pair ? sh.bn / 2 : sh.bn) * kBK * 2;
  sh.occ = (want_occ2 && (!sh.pair || g_occ2 == 1) && (kOcc2Smem - 1024 - kBarBytes) / sh.stage_bytes >= 3) ? 2 : 1;
  const int budget = sh.occ == 2 ? kOcc2Smem - 1024 - kBarBytes : kSmemBudget;
  int stages = (budget - extra_smem) / sh.stage_bytes;
  stages = stages > kMaxStages ? kMaxStages : stages;
  if (g_stage_cap > 0 && g_stage_cap < stages) stages = g_stage_cap;
  sh.stages = stages;
  sh.smem = 1024 + stages * sh.stage_bytes + kBarBytes + extra_smem;
  sh.slots = device_sms() * sh.occ;
  if (sh.pair) {
    sh.slots = max_pair_slots(sh.smem, sh.occ);
    if (sh.slots <= 0) return shape_for(T, N, K, extra_smem, true);  // no co-resident pair fits: single-CTA kernel
  }
  return sh;
}

struct Plan {
  bool balanced;
  int splits;       // uniform: K splits
  int slots;        // CTAs (pairs) launched
  int n_slices;     // partial slices written
  long long total;  // balanced: (tiles - dp) * kbt items of the stream-K tail
  int dp = 0;       // balanced: leading whole-K tiles (whole waves, data-parallel)
  int tail_slots = 0;
};

// Persistent CTAs (pairs) each stream their share of the weights; a step
// costs the busiest slot's bytes:
//   uniform(s): ceil(tiles*s/slots) units x (W slab / s + partial tile out)
//   balanced  : dp/slots whole-K units + ceil(total/tail_slots) k-blocks of
//               the tail, plus the partial tiles out
// Slices are capped so the callers' workspaces (max_slices slices) hold them.
Plan plan_for(const Shape& sh, int T, int N, int K, int max_slices) {
  const int tiles = ((N + sh.rows - 1) / sh.rows) * ((T + sh.unit_t - 1) / sh.unit_t);
  const int kbt = (K + kBK - 1) / kBK;
  const double w_kb = double(kBM) * kBK * 2.0;  // bytes of W one CTA streams per k-block
  // a partial tile is written here and re-read from L2 by the consumer: count the write
  const double out_tile = double(sh.unit_t) * kBM * 4.0;
  Plan best{false, 1, 0, 1, 0};
  double best_cost = 1e300;
  for (int s = 1; s <= max_slices && s <= 8 && kbt / s >= 4; ++s) {
    const int units = tiles * s;
    const int rounds = (units + sh.slots - 1) / sh.slots;
    const double cost = rounds * (w_kb * ((kbt + s - 1) / s) + out_tile);
    if (cost < best_cost * 0.97) {  // prefer fewer partial slices unless clearly better
      best_cost = cost;
      best = Plan{false, s, units < sh.slots ? units : sh.slots, s, 0};
    }
  }
  // auto: the balanced partition for decode-size steps of the short-K
  // projections (pure stream-K), and for > 512-row steps as whole waves of
  // whole-K tiles plus a stream-K tail when that beats the uniform splits
  // (wave quantization: o / down at T=1224-1736 lost 10-25% to it). Uniform
  // units keep the token tiles of one weight tile in step, so its weights
  // stream from HBM once and from L2 for the other tiles; a pure stream-K
  // partition of a many-token-tile step loses that (qkv at T=4096: 173 vs
  // 157 us) -- the data-parallel waves keep it for all but the tail.
  // tools/gemm_mixed.py: uniform measured faster than pure stream-K for
  // gate|up at T=712 (160 -> 138 us) and down at T=200-456 (4-7%).
  // Two-sub-tile units of the wide short-K projection (gate|up of a 257-512-row
  // mixed step: 112 pair tiles on 74 pairs) take one whole wave + a stream-K
  // tail too (tools/ab_sched.sh: T=328 73.7 -> 70.5 us, T=456 91.1 -> 88.3 us;
  // the narrow projections and the long-K down keep uniform splits)
  const bool wide_sub = sh.n_sub > 1 && K < kSubPairMinK && (N + kBM - 1) / kBM >= kPairMinTilesPerSm * device_sms();
  const bool auto_bal = (sh.n_sub == 1 && T <= kMaxBN && K < kSubPairMinK) || T > 2 * kMaxBN || wide_sub;
  if (g_sched != 0 && max_slices >= 2 && (g_sched == 1 || auto_bal)) {
    const int dp = T > kMaxBN ? (tiles / sh.slots) * sh.slots : 0;
    const long long total = (long long)(tiles - dp) * kbt;
    // a multi-token-tile step without one whole wave stays uniform: a pure
    // stream-K cut of it loses the weight reuse through L2 (down at T=1024:
    // 116 -> 129 us)
    if (total > 0 && !(T > kMaxBN && dp == 0)) {
      long long ts = total < sh.slots ? total : sh.slots;
      // a tail tile may touch at most max_slices ranges: share >= kbt / (max_slices - 1)
      ts = std::min(ts, (long long)(tiles - dp) * (max_slices - 1));
      const int tslots = (int)std::max(1LL, ts);
      const long long share = (total + tslots - 1) / tslots;
      // slices = most ranges touching one tile; segments = most tiles one range touches
      GemmParts g;
      g.kbt = kbt;
      g.slots = tslots;
      g.total = total;
      int n_slices = 1;
      for (long long t = 0; t < tiles - dp; ++t) {
        const int v = g.owner(t * kbt + kbt - 1) - g.owner(t * kbt) + 1;
        n_slices = v > n_slices ? v : n_slices;
      }
      const long long segs = (share + kbt - 1) / kbt + 1;
      const int dp_rounds = dp / sh.slots;
      const double cost = w_kb * (double(dp_rounds) * kbt + share) + (dp_rounds + segs) * out_tile;
      const bool want = g_sched == 1 || cost < best_cost * (T > kMaxBN ? 0.97 : 0.95);
      if (want && n_slices <= max_slices) {
        best = Plan{true, 1, dp > 0 ? sh.slots : tslots, n_slices, total, dp, tslots};
        best_cost = cost;
      }
    }
  }
  return best;
}

}  // namespace

int gemm_tc_plan_splits(int T, int N, int K) {
  const Shape sh = shape_for(T, N, K);
  const int cap = 8 * 256 / (T > 0 ? T : 1);
  const int saved = g_sched;
  g_sched = 0;
  const Plan pl = plan_for(sh, T, N, K, cap < 1 ? 1 : cap);
  g_sched = saved;
  return pl.splits;
}

namespace {

cudaError_t launch(const Shape& sh, const Plan& pl, const bf16* X, const bf16* W, void* out, int T, int N, int K,
                   bool out_f32, size_t split_stride, cudaStream_t s, int epi = kEpiPlain) {
  if (sh.stages < 2) return cudaErrorInvalidValue;  // ring does not fit
  GemmTcParams p{};
  p.out = out;
  p.T = T;
  p.N = N;
  p.K = K;
  p.ldo = epi == kEpiSilu ? N / 2 : N;
  p.epi = epi;
  p.bn = sh.bn;
  p.n_sub = sh.n_sub;
  p.out_f32 = out_f32 ? 1 : 0;
  p.splits = pl.balanced ? 1 : pl.splits;
  p.split_stride = split_stride ? split_stride : (size_t)T * N;
  // accumulator columns per segment (power of two >= bn); two accumulators when they fit
  p.bn_cols = sh.bn <= 32 ? 32 : sh.bn <= 64 ? 64 : sh.bn <= 128 ? 128 : 256;
  p.tmem_cols = 2 * sh.n_sub * p.bn_cols <= 512 ? 2 * sh.n_sub * p.bn_cols : sh.n_sub * p.bn_cols;
  if (sh.occ == 2) p.tmem_cols = p.bn_cols;  // two CTAs share the SM's 512 columns
  p.stages = sh.stages;
  p.balanced = pl.balanced ? 1 : 0;
  p.slots = pl.slots;
  p.total = pl.total;
  p.dp = pl.dp;
  p.tail_slots = pl.tail_slots;
  // weight-streaming shapes (<= 512 token rows) prefetch ahead into L2
  p.l2_pre = g_l2_pre >= 0 ? g_l2_pre : (T <= 2 * kMaxBN ? kL2PreAuto : 0);
  p.overlap = pdl_overlap();
  p.epi_pipe = g_epi_pipe ? 1 : 0;
  // evict-first only when every weight tile is read once (one token unit): with
  // several token tiles the other tiles re-read it from L2 (tools/ab_hint.sh:
  // B=16 / 64 decode steps -3.8% / -4.0%, B=200 -0.9%, 1536-token mix +0.8%)
  p.l2_hint = ((g_l2_hint & 1) && T <= sh.unit_t) ? 1 : 0;
  CUtensorMap mw, mx;
  if (!get_map(&mw, W, N, K, kBM) || !get_map(&mx, X, T, K, sh.pair ? sh.bn / 2 : sh.bn))
    return cudaErrorInvalidValue;
  set_smem_attrs();
  const GemmKernel kern = pick_kernel(sh.pair, epi, sh.occ, sh.n_sub);
  if (!kern) return cudaErrorInvalidValue;
  if (sh.pair)
    return launch_pdl_cluster(kern, dim3(2 * pl.slots), dim3(kThreads), (size_t)sh.smem, 2, s, mw, mx, p);
  return launch_pdl(kern, dim3(pl.slots), dim3(kThreads), (size_t)sh.smem, s, mw, mx, p);
}

}  // namespace

cudaError_t gemm_tc_run(const bf16* X, const bf16* W, void* out, int T, int N, int K, bool out_f32, int splits,
                        size_t split_stride, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  if (K % 8 != 0) return cudaErrorInvalidValue;  // TMA row stride must be 16 B aligned
  if (splits < 1) splits = 1;
  if (splits > 1 && !out_f32) return cudaErrorInvalidValue;
  const Shape sh = shape_for(T, N, K);
  const int tiles = ((N + sh.rows - 1) / sh.rows) * ((T + sh.unit_t - 1) / sh.unit_t);
  const int units = tiles * splits;
  const Plan pl{false, splits, units < sh.slots ? units : sh.slots, splits, 0};
  return launch(sh, pl, X, W, out, T, N, K, out_f32, split_stride, s);
}

cudaError_t gemm_tc_run_parts(const bf16* X, const bf16* W, float* out, int T, int N, int K, int max_slices,
                              size_t split_stride, GemmParts* parts, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  if (K % 8 != 0 || max_slices < 1) return cudaErrorInvalidValue;
  const Shape sh = shape_for(T, N, K);
  const Plan pl = plan_for(sh, T, N, K, max_slices);
  GemmParts g;
  g.n = pl.n_slices;
  g.stride = split_stride ? split_stride : (size_t)T * N;
  g.kbt = pl.balanced ? (K + kBK - 1) / kBK : 0;
  g.slots = pl.balanced ? pl.tail_slots : pl.slots;
  g.rows = sh.rows;
  g.bn = sh.unit_t;
  g.n_tiles_t = (T + sh.unit_t - 1) / sh.unit_t;
  g.total = pl.balanced ? pl.total : 1;
  g.dp = pl.balanced ? pl.dp : 0;
  *parts = g;
  return launch(sh, pl, X, W, out, T, N, K, true, g.stride, s);
}

cudaError_t gemm_tc_run_silu(const bf16* X, const bf16* W, bf16* m, int T, int N, int K, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  if (K % 8 != 0 || N % kBM != 0) return cudaErrorInvalidValue;  // whole gate|up groups per 128-row slab
  const Shape sh = shape_for(T, N, K, kXchgBytes);
  const int tiles = ((N + sh.rows - 1) / sh.rows) * ((T + sh.unit_t - 1) / sh.unit_t);
  const Plan pl{false, 1, tiles < sh.slots ? tiles : sh.slots, 1, 0};
  return launch(sh, pl, X, W, m, T, N, K, false, 0, s, kEpiSilu);
}

}  // namespace ppdk
