// layer_tc.cu — K8: the decode layer kernel. One persistent launch per layer
// for steps of <= 256 token rows (the decode step, the serving hot loop):
//
//   job 0  o-proj        attn[T][qd]  . Wo^T      -> proj32 slices
//   glue A               x += o ; h = RMSNorm(x)
//   job 1  gate|up       h[T][d]      . Wgu^T     -> gu32 slices
//   glue B               m = SiLU(gate) * up
//   job 2  down          m[T][F]      . Wdown^T   -> down32 slices
//   glue C               x += down ; h = RMSNorm(x)
//   job 3  next qkv      h[T][d]      . Wqkv'^T   -> qkv32 slices   (not after the last layer)
//   glue D               RoPE(q, k) ; paged K/V write of the next layer
//
// Why: a decode step is HBM-bound weight streaming (448 MB of weights per
// Llama-3-8B layer), and as four separate GEMM launches each one paid a
// fill (first TMA round trip) and a drain (epilogue tail, partially idle
// SMs), with the small ops between them on an idle HBM pipe. Here the weight
// stream never stops: the single TMA-producer thread of each CTA issues the
// next job's weights into free ring slots (and L2 prefetches beyond them)
// while the grid waits for a glue phase; only the activation half of a ring
// stage waits for the glue. The glue itself runs on the 8 epilogue warps of
// every CTA after a grid-wide counter barrier.
//
// Per CTA (384 threads, 1 per SM, grid = #SMs, all co-resident): warp 0 TMA
// producer, warp 1 single-thread tcgen05.mma issuer (M=128 weight rows x
// N=bn tokens, fp32 accumulators in TMEM, two alternating accumulators),
// warp 2 TMEM allocator, warps 4-11 epilogue (tcgen05.ld, warp w owns TMEM
// lanes 32*(w%4), column half (w-4)/4) and glue. Each GEMM is a stream-K
// partition: CTA c owns the contiguous (weight tile, k-block) items
// [c*total/ts, (c+1)*total/ts) and writes one fp32 partial slice per tile it
// touches (GemmParts rule, read back in slice order by the glue: the same
// deterministic sums as the stand-alone kernels' consumers).
//
// Grid barrier: per-step counters (zeroed by a memset node) — a CTA's
// epilogue warps arrive once per job when its partial slices are written
// (__threadfence + atomicAdd, release), the glue waits for n_cta arrivals
// (ld.acquire.gpu) and arrives on the glue-done counter the producer polls
// before loading the next job's activations (acquire + fence.proxy.async:
// the generic-proxy glue stores become visible to the TMA reads).
// Co-residency is required: the launcher is only used when the device is
// driven by ONE node (device.cu), and a waiting thread traps instead of
// hanging if a peer CTA never arrives.
//
// Status: an OPTION (tuning "layer_kernel", default off). Parity-green, but
// measured slower than the per-op path (Llama-3-8B shape, ctx 1024: B=200
// 12.7 vs 9.9 ms/step, B=64 9.6 vs 7.7, B=16 7.3 vs 5.7). The per-CTA
// event timeline (one layer, B=200) shows why: each job's main loop streams
// at the same ~27 GB/s per SM as the stand-alone single-CTA GEMM (gate|up
// 60 us vs 51-53 us for the CTA-pair GEMM), and every job boundary costs a
// ~6 us epilogue drain (100 KB of fp32 partials per CTA) + ~2 us of grid
// barrier during which the tensor cores idle — at B=200 the GEMMs sit at
// 78% of the tensor/HBM ridge, so idle MMA time is not hidden by the weight
// prefetch. DESIGN.md §9 has the numbers.
#include <cuda.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "ops_dev.cuh"
#include "tc_common.cuh"

namespace ppdk {

namespace {

constexpr int kThreadsL = 384;
constexpr int kBK = 64;                 // K elements per stage (128 B rows)
constexpr int kBM = 128;                // weight rows per tile (UMMA M)
constexpr int kWBytes = kBM * kBK * 2;  // 16 KB of weights per stage
constexpr int kMaxBN = 256;
constexpr int kMaxStagesL = 8;
constexpr int kBarBytesL = 256;
constexpr int kRedBytes = 256;          // glue block reductions
constexpr int kMaxTiles = 512;          // 128-column weight tiles per job (slice-count table)
constexpr int kSmemCap = 227 * 1024;
constexpr int kGlueThreads = 256;       // warps 4-11
constexpr int kNormChunks = 4;          // d_model <= 256 * 8 * 4
enum { kGlueAddNorm = 0, kGlueSilu = 1, kGlueRope = 2 };

// counter polls: relaxed gpu-scope loads (an ld.acquire.gpu per poll would
// invalidate L1 each time); one fence after the count is reached acquires
PPD_DEV unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
PPD_DEV void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
// release arrival: the caller's (and, through the preceding CTA barrier, its
// block's) global writes are visible before the count
PPD_DEV void arrive_release(unsigned* p) {
  __threadfence();
  atomicAdd(p, 1u);
}
// spin until *p >= target, then acquire; a peer CTA that never arrives is a
// bug, not a wait: trap after ~20 s of clock instead of hanging the GPU
PPD_DEV void wait_count(const unsigned* p, unsigned target) {
  const long long t0 = clock64();
  while (ld_relaxed(p) < target) {
    __nanosleep(32);
    if (clock64() - t0 > 40000000000LL) __trap();
  }
  __threadfence();
}
// non-blocking probe of an mbarrier phase (try_wait may suspend the thread)
PPD_DEV bool mbar_test(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
PPD_DEV void tma_prefetch_l2(const CUtensorMap* map, int x, int y) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y)
               : "memory");
}

PPD_DEV void job_range(const LayerParams& p, int j, int c, int& x, int& e) {
  const LayerJob& J = p.job[j];
  if (c < J.ts) {
    x = (int)((long long)c * J.total / J.ts);
    e = (int)((long long)(c + 1) * J.total / J.ts);
  } else {
    x = e = 0;
  }
}

// Walks this CTA's stream-K items of the jobs in order, one ring stage each.
// Incremental (tile, k-block): the single producer / MMA threads must not
// spend a division per stage (they are the per-SM issue path).
struct Cursor {
  int job, x, end, tile, kb, kbt;
  PPD_DEV void init(const LayerParams& p, int c) {
    job = -1;
    next_job(p, c);
  }
  PPD_DEV void next_job(const LayerParams& p, int c) {
    do {
      if (++job >= p.n_jobs) return;
      job_range(p, job, c, x, end);
    } while (x >= end);
    kbt = p.job[job].kbt;
    tile = x / kbt;
    kb = x - tile * kbt;
  }
  PPD_DEV bool valid(const LayerParams& p) const { return job < p.n_jobs; }
  // last k-block of its (tile) segment
  PPD_DEV bool seg_last() const { return x + 1 == end || kb + 1 == kbt; }
  PPD_DEV void next(const LayerParams& p, int c) {
    if (++x >= end) {
      next_job(p, c);
    } else if (++kb == kbt) {
      kb = 0;
      ++tile;
    }
  }
};

PPD_DEV const CUtensorMap* wmap(const LayerParams& p, int j) {
  return reinterpret_cast<const CUtensorMap*>(p.map_w[j]);
}
PPD_DEV const CUtensorMap* xmap(const LayerParams& p, int j) {
  return reinterpret_cast<const CUtensorMap*>(p.map_x[j]);
}

PPD_DEV int glue_kind(int j) { return j == 1 ? kGlueSilu : j == 3 ? kGlueRope : kGlueAddNorm; }

// ---- glue phases (warps 4-11; et = 0..255) --------------------------------
// nsl[t] = valid K-partial slices of the job's 128-column weight tile t (a
// smem table built at glue start: GemmParts::valid costs 64-bit divisions,
// which made the glue instruction-bound when evaluated per element).

// x += sum of the job's delta slices; h = RMSNorm(x), for rows c and c + n_cta.
// 256 threads per row: the sum of squares is reduced in a different order from
// add_rmsnorm_kernel's (one chunk per thread at d <= 4096), so inv_rms may
// differ in the last fp32 bit (the K8 tests compare within tolerance).
PPD_DEV void glue_add_norm(const LayerParams& p, const LayerJob& J, int c, int et, float* red, const uint8_t* nsl) {
  const int d = p.d_model, nc = d / 8;
  const int warp = et >> 5, lane = et & 31;
  for (int row = c; row < p.T; row += p.n_cta) {
    float v[kNormChunks][8];
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < kNormChunks; ++k) {
      const int cc = et + k * kGlueThreads;
      if (cc < nc) {
        unpack8(__ldcg(reinterpret_cast<const uint4*>(p.x + (size_t)row * d) + cc), v[k]);
        add_delta8<true, 4>(v[k], J.out, J.parts.stride, nsl[(cc * 8) >> 7], (size_t)row, d, cc);
        reinterpret_cast<uint4*>(p.x + (size_t)row * d)[cc] = pack8(v[k]);
#pragma unroll
        for (int j = 0; j < 8; ++j) ss += v[k][j] * v[k][j];
      }
    }
    ss = warp_sum(ss);
    if (lane == 0) red[warp] = ss;
    named_barrier_sync(1, kGlueThreads);
    float r = lane < 8 ? red[lane] : 0.f;
    r = warp_sum(r);
    const float inv = rms_inv(r, d, p.eps);
    named_barrier_sync(1, kGlueThreads);  // red[] is reused by the next row
#pragma unroll
    for (int k = 0; k < kNormChunks; ++k) {
      const int cc = et + k * kGlueThreads;
      if (cc < nc) reinterpret_cast<uint4*>(p.h + (size_t)row * d)[cc] = norm8(v[k], inv, p.norm_w, cc);
    }
  }
}

// four units per thread per round, all their slice loads in flight together
PPD_DEV void glue_silu(const LayerParams& p, const LayerJob& J, int c, int et, const uint8_t* nsl) {
  const int per_row = p.F / 4;
  const int n = p.T * per_row;
  const int stride = p.n_cta * kGlueThreads;
  for (int u0 = c * kGlueThreads + et; u0 < n; u0 += 4 * stride) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int u = u0 + i * stride;
      if (u < n) {
        const int r = u / per_row, j = (u - r * per_row) * 4;
        silu4<true>(J.out, J.parts.stride, nsl[j >> 6], p.m, p.F, r, j);
      }
    }
  }
}

PPD_DEV void glue_rope(const LayerParams& p, int c, int et, const uint8_t* nsl) {
  const int per_row = rope_units_per_row(p.rope);
  const int n = p.T * per_row;
  const int stride = p.n_cta * kGlueThreads;
  for (int u0 = c * kGlueThreads + et; u0 < n; u0 += 2 * stride) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int u = u0 + i * stride;
      if (u < n) {
        const int r = u / per_row, ur = u - r * per_row;
        rope_kv_unit<true, 2>(p.rope, r, ur, nsl[rope_unit_col(p.rope, ur) >> 7]);
      }
    }
  }
}

}  // namespace

__global__ void __launch_bounds__(kThreadsL, 1) decode_layer_kernel(const __grid_constant__ LayerParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = p.stages, SB = p.stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * SB);
  uint64_t* empty = full + S;
  uint64_t* acc_full = empty + S;      // [2]
  uint64_t* acc_empty = acc_full + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  float* red = reinterpret_cast<float*>(smem + S * SB + kBarBytesL);
  uint8_t* nsl = smem + S * SB + kBarBytesL + kRedBytes;  // [kMaxTiles] slice counts of the glue's job

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x;
  const int acc_cols = p.bn <= 128 ? 128 : 256;

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 8);  // one arrive per epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == 2) tc::alloc(tmem_slot, 2 * acc_cols);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer: three cursors over the same stage sequence ----
      // w: weights (slot free), a: activations (job inputs ready), pf: L2 prefetch
      const uint32_t tx = (uint32_t)(kWBytes + p.bn * kBK * 2);
      Cursor w, a, pf;
      w.init(p, c);
      a = w;
      pf = w;
      int wi = 0, ai = 0, pi = 0, ready = -1;
      auto issue_w = [&]() {
        const int s = wi % S;
        mbar_arrive_expect_tx(&full[s], tx);
        tc::tma_load_2d(smem + s * SB, wmap(p, w.job), w.kb * kBK, w.tile * kBM, &full[s]);
        w.next(p, c);
        ++wi;
      };
      // the predecessor (attention) does not write weights: fill the ring first
      while (w.valid(p) && wi < S) issue_w();
      pdl_wait();
      pdl_trigger();
      ready = 0;
      // The loop never blocks on one resource while another could progress:
      // every activation whose weights are issued and whose job is ready goes
      // out first (a blocking wait on a ring slot here would serialise the
      // activation loads behind the MMAs), then a free slot (non-blocking
      // probe) takes the next weights, else the L2 prefetch runs ahead.
      while (a.valid(p)) {
        while (ai < wi) {
          if (a.job > ready) {
            if (ld_relaxed(p.sync + 2 * (a.job - 1) + 1) < (unsigned)p.n_cta) break;
            __threadfence();             // acquire the glue's stores
            fence_proxy_async_global();  // ... for our TMA (async proxy) reads
            ready = a.job;
          }
          const int s = ai % S;
          tc::tma_load_2d(smem + s * SB + kWBytes, xmap(p, a.job), a.kb * kBK, 0, &full[s]);
          a.next(p, c);
          ++ai;
        }
        if (!a.valid(p)) break;
        if (w.valid(p) && wi < ai + S && mbar_test(&empty[wi % S], ((wi / S) - 1) & 1)) {
          issue_w();
          continue;
        }
        // nothing to issue: keep HBM busy with the weights beyond the ring
        if (pi < wi) {
          pf = w;
          pi = wi;
        }
        if (pf.valid(p) && pi < wi + p.l2_ahead) {
          tma_prefetch_l2(wmap(p, pf.job), pf.kb * kBK, pf.tile * kBM);
          pf.next(p, c);
          ++pi;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---- MMA issuer ----
      const uint32_t idesc = tc::idesc_bf16(kBM, p.bn, false);
      Cursor cu;
      cu.init(p, c);
      int it = 0, seg = 0;
      while (cu.valid(p)) {
        const int acc = seg & 1, use = seg >> 1;
        if (use > 0) mbar_wait(&acc_empty[acc], (use - 1) & 1);
        tc::fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * acc_cols);
        bool first = true, last;
        do {
          const int s = it % S;
          mbar_wait(&full[s], (it / S) & 1);
          tc::fence_after();
          const uint32_t sa = smem_u32(smem + s * SB);
          const uint64_t da = tc::desc_kmajor_sw128(sa), db = tc::desc_kmajor_sw128(sa + kWBytes);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
            tc::mma_bf16_ss(d_tmem, da + (uint64_t)(k * 2), db + (uint64_t)(k * 2), idesc, (!first) || (k != 0));
          tc::commit(&empty[s]);
          last = cu.seg_last();
          cu.next(p, c);
          ++it;
          first = false;
        } while (!last);
        tc::commit(&acc_full[acc]);
        ++seg;
      }
    }
  } else if (warp >= 4) {
    // ---- epilogue + glue (256 threads) ----
    pdl_wait();
    const int et = threadIdx.x - 128;
    const int q = warp & 3, hh = (warp - 4) >> 2;
    int seg = 0;
    for (int j = 0; j < p.n_jobs; ++j) {
      const LayerJob& J = p.job[j];
      int x, e;
      job_range(p, j, c, x, e);
      while (x < e) {
        const int tile = x / J.kbt;
        const int seg_end = min(e, (tile + 1) * J.kbt);
        const int slice = c - J.parts.owner((long long)tile * J.kbt);
        const int acc = seg & 1, use = seg >> 1;
        mbar_wait(&acc_full[acc], use & 1);
        tc::fence_after();
        const int row = tile * kBM + q * 32 + lane;
        float* out = J.out + (size_t)slice * J.parts.stride;
        const uint32_t t_acc = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * acc_cols);
        for (int c0 = hh * 32; c0 < p.T; c0 += 64) {
          uint32_t r[32];
          tc::ld32x32(t_acc + (uint32_t)c0, r);
          tc::wait_ld();
          if (row < J.N) {
            const int nj = min(32, p.T - c0);
            float* dst = out + (size_t)c0 * J.N + row;
#pragma unroll
            for (int jj = 0; jj < 32; ++jj)
              if (jj < nj) dst[(size_t)jj * J.N] = __uint_as_float(r[jj]);
          }
        }
        tc::fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[acc]);
        x = seg_end;
        ++seg;
      }
      // this CTA's partial slices of job j are written
      named_barrier_sync(1, kGlueThreads);
      if (et == 0) {
        arrive_release(p.sync + 2 * j);
        wait_count(p.sync + 2 * j, (unsigned)p.n_cta);
      }
      for (int t = et; t < J.N / kBM; t += kGlueThreads) nsl[t] = (uint8_t)J.parts.valid(t * kBM, 0);
      named_barrier_sync(1, kGlueThreads);
      const int g = glue_kind(j);
      if (g == kGlueAddNorm)
        glue_add_norm(p, J, c, et, red, nsl);
      else if (g == kGlueSilu)
        glue_silu(p, J, c, et, nsl);
      else
        glue_rope(p, c, et, nsl);
      named_barrier_sync(1, kGlueThreads);
      if (et == 0) arrive_release(p.sync + 2 * j + 1);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 2) tc::dealloc(tmem_base, 2 * acc_cols);
}

// ----------------------------------------------------------------- host side
bool layer_plan_job(LayerJob& j, float* out, int T, int N, int K, int n_cta, int max_slices) {
  if (N % kBM != 0 || K % kBK != 0 || N / kBM > kMaxTiles) return false;
  max_slices = std::min(max_slices, kMaxSlices);
  j.out = out;
  j.N = N;
  j.K = K;
  j.kbt = K / kBK;
  const int tiles = N / kBM;
  j.total = (long long)tiles * j.kbt;
  // a range of >= kbt / (max_slices - 1) items: a tile meets at most max_slices ranges
  j.ts = (int)std::min<long long>({(long long)n_cta, j.total, (long long)tiles * std::max(1, max_slices - 1)});
  GemmParts g;
  g.kbt = j.kbt;
  g.slots = j.ts;
  g.total = j.total;
  g.rows = kBM;
  g.bn = kMaxBN;  // one token tile
  g.n_tiles_t = 1;
  g.dp = 0;
  g.stride = (size_t)T * N;
  int n_slices = 1;
  for (int t = 0; t < tiles; ++t) {
    const int v = g.owner((long long)t * j.kbt + j.kbt - 1) - g.owner((long long)t * j.kbt) + 1;
    n_slices = std::max(n_slices, v);
  }
  g.n = n_slices;
  j.parts = g;
  return n_slices <= max_slices;
}

void layer_shape(int T, int* bn, int* stages, int* stage_bytes, int* smem) {
  *bn = ((T + 15) / 16) * 16;
  *stage_bytes = kWBytes + *bn * kBK * 2;
  const int budget = kSmemCap - 1024 - kBarBytesL - kRedBytes - kMaxTiles;
  *stages = T <= kMaxBN ? std::min(kMaxStagesL, budget / *stage_bytes) : 0;
  *smem = 1024 + *stages * *stage_bytes + kBarBytesL + kRedBytes + kMaxTiles;
}

cudaError_t launch_decode_layer(const LayerParams& p, int smem, cudaStream_t s) {
  static unsigned long long done_devs = 0;
  if (first_on_device(&done_devs))
    cudaFuncSetAttribute(decode_layer_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemCap);
  if (p.stages < 2 || p.T > 2 * p.n_cta || p.d_model > kGlueThreads * 8 * kNormChunks) return cudaErrorInvalidValue;
  return launch_pdl(decode_layer_kernel, dim3(p.n_cta), dim3(kThreadsL), (size_t)smem, s, p);
}

}  // namespace ppdk
