// attention_tc_body.cuh — the K3/K4 tcgen05 prefill tile (full / append
// prefill attention over the paged pool), shared by the standalone kernel
// (attention_tc.cu, one CTA per tile) and the fused mixed decode + prefill
// launch (attention.cu, mixed_attention_kernel: prefill CTAs loop over tiles).
// See attention_tc.cu for the warp roles.
#pragma once
#include <cuda.h>

#include "kernels.h"
#include "tc_common.cuh"

namespace ppdk {
namespace pftc {

// warps 0-3: K TMA / MMA / TMEM alloc / V TMA; warps 4.. : kSW softmax warps,
// kSW / 4 threads per query row (8: 64 key columns each, 16: 32 each)
constexpr int threads_for(int kSW) { return 128 + 32 * kSW; }
constexpr int kBT = 16;
constexpr int kDh = 128;
constexpr int kKeys = 128;                  // keys per block
constexpr int kTile = 32768;                // 128 x 128 bf16
// P_j (bf16) is written back into S_j's own TMEM columns and PV_j takes its A
// operand from TMEM (FA4-style aliasing): no shared-memory P buffers, no
// st.shared / proxy fence per block. S_{j+2} reuses the columns only after
// PV_j in the MMA pipe's issue order (tcgen05.mma from one thread executes in
// order). kPInTmem = false keeps the double-buffered shared-memory P (A/B).
#ifndef PPD_PF_P_SMEM
constexpr bool kPInTmem = true;
#else
constexpr bool kPInTmem = false;
#endif
#ifndef PPD_PF_KSTAGES
constexpr int kKStages = 2;  // K ring: released as soon as S_j retires
#else
constexpr int kKStages = PPD_PF_KSTAGES;
#endif
#ifndef PPD_PF_VSTAGES
constexpr int kVStages = 2;  // V ring: released after PV_j
#else
constexpr int kVStages = PPD_PF_VSTAGES;
#endif
constexpr int kPBufs = kPInTmem ? 0 : 2;
// the parts of a query row agree on the running max (and, at the end, the row
// sum) through shared memory (one st.shared + a 32 NH-thread named barrier +
// NH ld.shared); kXchgSmem = false uses free TMEM columns instead (A/B)
#ifndef PPD_PF_XCHG_TMEM
constexpr bool kXchgSmem = true;
#else
constexpr bool kXchgSmem = false;
#endif
constexpr int kXchgBytes = 3 * 128 * 4 * 4;  // [3 slots: max parity 0/1, row sum][128 rows][NH <= 4]
constexpr int kSmem = 1024 + kTile /*Q*/ + (kKStages + kVStages) * kTile + kPBufs * kTile /*P*/ + 256 + kXchgBytes;
constexpr uint32_t kTmemCols = 512;        // S0 | S1 | O | S2 (or the TMEM max exchange, cols 384..)
constexpr uint32_t kXchgCol = 384;
constexpr float kRescaleThreshold = 8.0f;   // log2 domain
// S buffers in TMEM. Three (S0 | S1 | O | S2) when P lives in TMEM and the
// max exchange in shared memory: S_j is then issued two blocks ahead of PV_j,
// so softmax_{j+1}'s scores are ready when softmax_j ends (with two, S_{j+1}
// can only follow PV_{j-1}, and softmax waits out PV + S every other block).
constexpr int kSBufs = (kPInTmem && kXchgSmem) ? 3 : 2;
// diagnostics builds only (-DPPD_PF_DIAG=n, results wrong): 1 softmax without
// exponentials, 2 PV reduced to one K slice, 3 S reduced to one K slice, 4 half
// the S columns read from TMEM
#ifndef PPD_PF_DIAG
constexpr int kDiag = 0;
#else
constexpr int kDiag = PPD_PF_DIAG;
#endif
PPD_DEV constexpr uint32_t s_col(int b) { return b < 2 ? (uint32_t)b * kKeys : 3u * kKeys; }
constexpr int kNumBars = 2 * (kKStages + kVStages) + 2 * kSBufs + 3;
// one key pair in kPolyEvery goes to the FMA-pipe polynomial, the rest to MUFU.EX2
#ifndef PPD_PF_POLY_EVERY
constexpr int kPolyEvery = 8;
#else
constexpr int kPolyEvery = PPD_PF_POLY_EVERY;
#endif

PPD_DEV float ex2_sfu(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x = 2^n * p(x - n), n = round(x), p a minimax cubic on [-1/2, 1/2] with
// p(0) = 1 (max rel. error 1.0e-4 << bf16 ulp). Rounding by the 1.5 * 2^23
// magic add and the exponent insert by an integer add keep it entirely on the
// FMA / ALU pipes (FRND / F2I would share the SFU-class pipe with MUFU.EX2).
// Two lanes at a time: the float math issues as packed f32x2 FADD2 / FFMA2.
PPD_DEV float2 ex2_poly2(float2 x) {
  x.x = fmaxf(x.x, -126.f);  // -inf (masked keys) -> ~0
  x.y = fmaxf(x.y, -126.f);
  const float2 t = __fadd2_rn(x, make_float2(12582912.0f, 12582912.0f));
  const float2 u = __fadd2_rn(t, make_float2(-12582912.0f, -12582912.0f));  // round(x), exact
  const float2 f = __ffma2_rn(u, make_float2(-1.f, -1.f), x);                 // x - round(x), exact
  float2 p = __ffma2_rn(make_float2(0.05500893f, 0.05500893f), f, make_float2(0.24221098f, 0.24221098f));
  p = __ffma2_rn(p, f, make_float2(0.69328293f, 0.69328293f));
  p = __ffma2_rn(p, f, make_float2(1.0f, 1.0f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

// shared-memory carve-up of one prefill CTA (smem 1024-byte aligned)
struct Smem {
  uint8_t *q_s, *k_s, *v_s, *p_s;
  uint64_t *bars, *k_full, *k_empty, *v_full, *v_empty, *s_full, *p_ready, *o_done, *q_ready;
  uint32_t* tmem_slot;
  float* xchg;  // [3][128][NH]
  PPD_DEV explicit Smem(uint8_t* smem) {
    q_s = smem;
    k_s = smem + kTile;              // [kKStages]
    v_s = k_s + kKStages * kTile;    // [kVStages]
    p_s = v_s + kVStages * kTile;    // [kPBufs]
    bars = reinterpret_cast<uint64_t*>(p_s + kPBufs * kTile);
    k_full = bars;                  // [kKStages]
    k_empty = k_full + kKStages;    // [kKStages]
    v_full = k_empty + kKStages;    // [kVStages]
    v_empty = v_full + kVStages;    // [kVStages]
    s_full = v_empty + kVStages;    // [kSBufs]: S_j commits to s_full[j % kSBufs]
    p_ready = s_full + kSBufs;      // [kSBufs]: softmax_j arrives on p_ready[j % kSBufs]
    o_done = p_ready + kSBufs;      // [2]: PV_j commits to o_done[j & 1]
    q_ready = o_done + 2;
    tmem_slot = reinterpret_cast<uint32_t*>(bars + kNumBars);
    xchg = reinterpret_cast<float*>(p_s + kPBufs * kTile + 256);
  }
};

// one thread: (re)initialise the tile's mbarriers
template <int kSW>
PPD_DEV void init_barriers(const Smem& S, bool reinit) {
  if (reinit)
    for (int i = 0; i < kNumBars; ++i)
      asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(S.bars + i)) : "memory");
  for (int i = 0; i < kKStages; ++i) {
    mbar_init(&S.k_full[i], 1);
    mbar_init(&S.k_empty[i], 1);
  }
  for (int i = 0; i < kVStages; ++i) {
    mbar_init(&S.v_full[i], 1);
    mbar_init(&S.v_empty[i], 1);
  }
  for (int i = 0; i < kSBufs; ++i) mbar_init(&S.s_full[i], 1);
  for (int i = 0; i < kSBufs; ++i) mbar_init(&S.p_ready[i], kSW);
  for (int i = 0; i < 2; ++i) mbar_init(&S.o_done[i], 1);
  mbar_init(S.q_ready, kSW);
  fence_barrier_init();
}

// NH consecutive 32-bit TMEM columns of this thread's lane -> max / sum (fixed order)
template <int NH>
PPD_DEV void ld_cols(uint32_t taddr, float* v) {
  if constexpr (NH == 2) {
    uint32_t a, b;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(a), "=r"(b) : "r"(taddr));
    tc::wait_ld();
    v[0] = __uint_as_float(a);
    v[1] = __uint_as_float(b);
  } else {
    uint32_t a, b, c, d;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                 : "r"(taddr));
    tc::wait_ld();
    v[0] = __uint_as_float(a);
    v[1] = __uint_as_float(b);
    v[2] = __uint_as_float(c);
    v[3] = __uint_as_float(d);
  }
}
template <int NH>
PPD_DEV float xchg_max(uint32_t taddr) {
  float v[NH];
  ld_cols<NH>(taddr, v);
  float m = v[0];
#pragma unroll
  for (int i = 1; i < NH; ++i) m = fmaxf(m, v[i]);
  return m;
}
template <int NH>
PPD_DEV float xchg_sum(uint32_t taddr) {
  float v[NH];
  ld_cols<NH>(taddr, v);
  float s = v[0];
#pragma unroll
  for (int i = 1; i < NH; ++i) s += v[i];
  return s;
}

// One 128-row tile (128/G query tokens x the G query heads of kv head `kvh`)
// of prefill item `it`, run by warps 0..11 of the calling CTA. Barriers are
// freshly initialised; `tmem` holds kTmemCols columns (S0 | S1 | O).
template <int kSW>
PPD_DEV void tile(const CUtensorMap* kv_map, const AttnParams& p, const Smem& S, const AttnItem& it, int kvh,
                  uint32_t tmem, int warp, int lane, bool trigger_pdl) {
  uint8_t* q_s = S.q_s;
  uint8_t* k_s = S.k_s;
  uint8_t* v_s = S.v_s;
  uint8_t* p_s = S.p_s;
  uint64_t* k_full = S.k_full;
  uint64_t* k_empty = S.k_empty;
  uint64_t* v_full = S.v_full;
  uint64_t* v_empty = S.v_empty;
  uint64_t* s_full = S.s_full;
  uint64_t* p_ready = S.p_ready;
  uint64_t* o_done = S.o_done;
  uint64_t* q_ready = S.q_ready;
  const int G = p.group;
  const int s = it.seq;
  const int ctx = p.ctx[s];
  const int q_base = p.q_start[s];
  const int rows = it.n_q * G;
  const int key_end = ctx + it.q_tok0 + it.n_q;
  const int nblk = (key_end + kKeys - 1) / kKeys;
  const int* btab = p.block_tables + (size_t)s * p.max_blocks;

  const uint32_t t_o = tmem + 2 * kKeys;

  if (warp == 0 || warp == 3) {
    // warp 0 streams K, warp 3 streams V; the 16 TMA boxes of a 128-key tile
    // (8 paged blocks x two 64-dim halves) are issued by 16 lanes in parallel.
    const bool is_v = warp == 3;
    const int n_st = is_v ? kVStages : kKStages;
    uint64_t* fullb = is_v ? v_full : k_full;
    uint64_t* emptyb = is_v ? v_empty : k_empty;
    uint8_t* ring = is_v ? v_s : k_s;
    const int last_blk = (key_end - 1) / kBT;
    const int b = (lane >> 1) & 7, h = lane & 1;
    for (int j = 0; j < nblk; ++j) {
      const int st = j % n_st;
      if (j >= n_st) mbar_wait(&emptyb[st], ((j / n_st) - 1) & 1);
      if (lane == 0) mbar_arrive_expect_tx(&fullb[st], kTile);
      __syncwarp();
      if (lane < 16) {
        // slots past the sequence re-load its last block: finite data, masked to p = 0
        const int pb = min(j * (kKeys / kBT) + b, last_blk);
        const int blk = btab[pb];
        const int row = (((blk * p.n_layers + p.layer) * 2 + (is_v ? 1 : 0)) * p.n_kv_heads + kvh) * kBT;
        tc::tma_load_2d(ring + st * kTile + h * (kTile / 2) + b * 2048, kv_map, h * 64, row, &fullb[st]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id_s = tc::idesc_bf16(128, kKeys, false);
      const uint32_t id_o = tc::idesc_bf16(128, kDh, true);
      mbar_wait(q_ready, 0);
      tc::fence_after();
      const uint32_t qa = smem_u32(q_s), pa = smem_u32(p_s);
      constexpr int kAhead = kSBufs - 1;  // S_j is issued before PV_{j - kAhead}
      for (int j = 0; j < nblk + kAhead; ++j) {
        if (j < nblk) {
          const int st = j % kKStages;
          mbar_wait(&k_full[st], (j / kKStages) & 1);
          tc::fence_after();
          const uint32_t ka = smem_u32(k_s + st * kTile);
#pragma unroll
          for (int kk = 0; kk < kDh / 16; ++kk) {
            if (kDiag == 3 && kk > 0) break;  // diagnostics: one K=16 slice of S only
            const uint32_t off = (kk >> 2) * (kTile / 2) + (kk & 3) * 32;
            tc::mma_bf16_ss(tmem + s_col(j % kSBufs), tc::desc_kmajor_sw128(qa + off),
                            tc::desc_kmajor_sw128(ka + off), id_s, kk > 0);
          }
          tc::commit(&s_full[j % kSBufs]);
          tc::commit(&k_empty[st]);  // K tile free once S_j retires
        }
        if (j >= kAhead) {
          const int jj = j - kAhead, st = jj % kVStages;
          mbar_wait(&p_ready[jj % kSBufs], (jj / kSBufs) & 1);
          mbar_wait(&v_full[st], (jj / kVStages) & 1);
          tc::fence_after();
          const uint32_t va = smem_u32(v_s + st * kTile);
          if constexpr (kPInTmem) {
            // part h of a row packed its CPT keys into columns [CPT h, CPT h + CPT / 2) of S_jj
            constexpr int CPT = kKeys / (kSW / 4);
            const uint32_t sj = tmem + s_col(jj % kSBufs);
#pragma unroll
            for (int kk = 0; kk < kKeys / 16; ++kk) {
              if (kDiag == 2 && kk > 0) break;  // diagnostics: one K=16 slice of PV only
              const uint32_t col = (16 * kk / CPT) * CPT + ((16 * kk) % CPT) / 2;
              tc::mma_bf16_ts(t_o, sj + col, tc::desc_mnmajor_sw128(va + kk * 2048, kTile / 2), id_o,
                              (jj > 0) || (kk > 0));
            }
          } else {
            const uint32_t pj = pa + (uint32_t)((jj & 1) * kTile);
#pragma unroll
            for (int kk = 0; kk < kKeys / 16; ++kk) {
              const uint32_t poff = (kk >> 2) * (kTile / 2) + (kk & 3) * 32;
              tc::mma_bf16_ss(t_o, tc::desc_kmajor_sw128(pj + poff), tc::desc_mnmajor_sw128(va + kk * 2048, kTile / 2),
                              id_o, (jj > 0) || (kk > 0));
            }
          }
          tc::commit(&o_done[jj & 1]);
          tc::commit(&v_empty[st]);
        }
      }
    }
  } else if (warp >= 4) {
    // Softmax: kSW warps, NH = kSW / 4 threads per query row. Warp w handles
    // TMEM lane quarter w & 3 (row r) and key / O columns [CPT h, CPT (h+1)),
    // h = (w - 4) / 4. The parts of a row agree on its running max through
    // free TMEM columns (one tcgen05.st + one tcgen05.ld per block) and a
    // (32 NH)-thread named barrier per lane quarter; l is kept per part and
    // summed (fixed order) in the epilogue.
    constexpr int NH = kSW / 4, CPT = kKeys / NH;
    const int q4 = warp & 3;
    const int h = (warp - 4) >> 2;
    const int r = q4 * 32 + lane;  // query row == TMEM lane
    const uint32_t lane_base = (uint32_t)(q4 * 32) << 16;
    const int pair_bar = 8 + q4;
    // ---- Q row part -> shared (K-major, 128 B swizzle: atom c >> 3 holds dims [64 (c>>3), +64))
    {
      const uint4* src = nullptr;
      if (r < rows)
        src = reinterpret_cast<const uint4*>(p.q + ((size_t)(q_base + it.q_tok0 + r / G) * p.n_q_heads + kvh * G + r % G) * kDh);
#pragma unroll
      for (int c = (16 / NH) * h; c < (16 / NH) * (h + 1); ++c) {
        const uint4 v = src ? src[c] : make_uint4(0, 0, 0, 0);
        sts_u128(q_s + (c >> 3) * (kTile / 2) + r * 128 + (((c & 7) ^ (r & 7)) << 4), v);
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(q_ready);
    }
    const int pos = r < rows ? ctx + it.q_tok0 + r / G : -1;
    const float sl2 = p.scale_log2;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < nblk; ++j) {
      const int sb = j % kSBufs;
      mbar_wait(&s_full[sb], (j / kSBufs) & 1);
      tc::fence_after();
      uint32_t raw[CPT];
#pragma unroll
      if (kDiag == 4) {  // diagnostics: one 32-column TMEM load, replicated (S read cost removed)
        tc::ld32x32(tmem + lane_base + s_col(sb) + CPT * h, raw);
#pragma unroll
        for (int c = 32; c < CPT; ++c) raw[c] = raw[c - 32] ^ (uint32_t)c;
      } else {
#pragma unroll
        for (int c0 = 0; c0 < CPT; c0 += 32) tc::ld32x32(tmem + lane_base + s_col(sb) + CPT * h + c0, raw + c0);
      }
      tc::wait_ld();
      // raw (unscaled) scores; the scale folds into the exponent's FFMA below
      // (sl2 > 0: the max commutes with it)
      float sv[CPT];
      const int key0 = j * kKeys + CPT * h;
      float mxp[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mxp[i] = -INFINITY;
      if (key0 + CPT - 1 <= pos) {  // no causal mask inside this part of the block
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          sv[c] = __uint_as_float(raw[c]);
          mxp[c & 7] = fmaxf(mxp[c & 7], sv[c]);
        }
      } else {
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          sv[c] = (key0 + c <= pos) ? __uint_as_float(raw[c]) : -INFINITY;
          mxp[c & 7] = fmaxf(mxp[c & 7], sv[c]);
        }
      }
      const float mh = fmaxf(fmaxf(fmaxf(mxp[0], mxp[1]), fmaxf(mxp[2], mxp[3])),
                             fmaxf(fmaxf(mxp[4], mxp[5]), fmaxf(mxp[6], mxp[7]))) * sl2;
      // exchange the part maxima (parity-double-buffered slots: a part writes
      // slot j & 1 only after every part passed block j-1's barrier)
      float mx;
      if constexpr (kXchgSmem) {
        float* slot = S.xchg + ((j & 1) * 128 + r) * NH;
        sts_f32(slot + h, mh);
        named_barrier_sync(pair_bar, 32 * NH);
        mx = lds_f32(slot);
#pragma unroll
        for (int i = 1; i < NH; ++i) mx = fmaxf(mx, lds_f32(slot + i));  // identical in every part
      } else {
        uint32_t v = __float_as_uint(mh);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(
                         tmem + lane_base + kXchgCol + NH * (j & 1) + h),
                     "r"(v)
                     : "memory");
        tc::wait_st();
        tc::fence_before();
        named_barrier_sync(pair_bar, 32 * NH);
        tc::fence_after();
        mx = xchg_max<NH>(tmem + lane_base + kXchgCol + NH * (j & 1));  // identical in every part
      }
      float alpha = 1.f;
      bool rescale = false;
      if (m == -INFINITY) {
        m = mx;  // first keys this row sees (O holds zeros for it so far)
      } else if (mx > m + kRescaleThreshold) {
        alpha = exp2f(m - mx);
        m = mx;
        rescale = true;
      }
      const float base = m == -INFINITY ? 0.f : m;
      // exp2 on two pipes: of every 2 kPolyEvery keys, the last two go to a
      // degree-3 polynomial on the FMA pipe (max rel. error 8.6e-5 << bf16
      // ulp), the rest to the SFU (ex2.approx); scale, polynomial and row
      // sums as packed f32x2 ops
      const float2 sl2v = make_float2(sl2, sl2), nbase = make_float2(-base, -base);
      float2 rs_a = make_float2(0.f, 0.f), rs_b = make_float2(0.f, 0.f);
      uint32_t pk[CPT / 2];
#pragma unroll
      for (int c = 0; c < CPT; c += 2) {
        if (kDiag == 1) {  // diagnostics: no exponentials
          pk[c >> 1] = __float_as_uint(sv[c]) ^ __float_as_uint(sv[c + 1]);
          continue;
        }
        const float2 x = __ffma2_rn(make_float2(sv[c], sv[c + 1]), sl2v, nbase);
        float2 e;
        if ((c / 2) % kPolyEvery == kPolyEvery - 1) {
          e = ex2_poly2(x);
          rs_b = __fadd2_rn(rs_b, e);
        } else {
          e = make_float2(ex2_sfu(x.x), ex2_sfu(x.y));
          rs_a = __fadd2_rn(rs_a, e);
        }
        pk[c >> 1] = pack2(e.x, e.y);
      }
      const float rs = (rs_a.x + rs_a.y) + (rs_b.x + rs_b.y);
      if constexpr (kPInTmem) {
        // consume PV_{j-2}'s o_done phase (long retired; keeps every mbarrier
        // phase observed before its next arrival, as compute-sanitizer
        // synccheck requires), then P_j over this part's own (already loaded)
        // S_j columns; every part's S loads precede the max-exchange barrier above
        if (j >= 2) mbar_wait(&o_done[j & 1], ((j - 2) >> 1) & 1);
        const uint32_t pdst = tmem + lane_base + s_col(sb) + CPT * h;
        if constexpr (CPT == 32) {
          tc::st32x16(pdst, pk);
        } else {
          tc::st32x32(pdst, pk);
        }
      } else {
        // P buffer j & 1 was last read by PV_{j-2}
        if (j >= 2) {
          mbar_wait(&o_done[j & 1], ((j - 2) >> 1) & 1);
          tc::fence_after();
        }
        uint8_t* pbuf = p_s + (j & 1) * kTile;
#pragma unroll
        for (int cc = 0; cc < CPT / 8; ++cc) {
          const int c = (CPT / 8) * h + cc;  // 16-byte chunk of the row
          const uint4 v = make_uint4(pk[cc * 4], pk[cc * 4 + 1], pk[cc * 4 + 2], pk[cc * 4 + 3]);
          *reinterpret_cast<uint4*>(pbuf + (c >> 3) * (kTile / 2) + r * 128 + (((c & 7) ^ (r & 7)) << 4)) = v;
        }
      }
      if (j >= 1 && __any_sync(0xffffffffu, rescale)) {
        // O must hold PV_{j-1} before it is rescaled (rare: lazy threshold)
        mbar_wait(&o_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
        tc::fence_after();
#pragma unroll
        for (int c0 = CPT * h; c0 < CPT * (h + 1); c0 += 32) {
          uint32_t o[32];
          tc::ld32x32(t_o + lane_base + c0, o);
          tc::wait_ld();
#pragma unroll
          for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * alpha);
          tc::st32x32(t_o + lane_base + c0, o);
        }
        tc::wait_st();
      }
      l = l * alpha + rs;
      if constexpr (kPInTmem) {
        tc::wait_st();
      } else {
        fence_proxy_async();
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_ready[sb]);
    }
    // ---- epilogue: O / (l_0 + ... + l_{NH-1}) -> bf16, each part its CPT columns
    if (trigger_pdl) pdl_trigger();
    float lsum;
    if constexpr (kXchgSmem) {
      float* slot = S.xchg + (2 * 128 + r) * NH;
      sts_f32(slot + h, l);
      named_barrier_sync(pair_bar, 32 * NH);
      lsum = lds_f32(slot);
#pragma unroll
      for (int i = 1; i < NH; ++i) lsum += lds_f32(slot + i);  // same order in every part
    } else {
      uint32_t v = __float_as_uint(l);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + lane_base + kXchgCol + 2 * NH + h),
                   "r"(v)
                   : "memory");
      tc::wait_st();
      tc::fence_before();
      named_barrier_sync(pair_bar, 32 * NH);
      tc::fence_after();
      lsum = xchg_sum<NH>(tmem + lane_base + kXchgCol + 2 * NH);  // same order in every part
    }
    // the final phase of both o_done slots is consumed before the barriers are
    // re-armed for the next tile (PV_{nblk-2} retired before PV_{nblk-1})
    if (nblk >= 2) mbar_wait(&o_done[(nblk - 2) & 1], ((nblk - 2) >> 1) & 1);
    mbar_wait(&o_done[(nblk - 1) & 1], ((nblk - 1) >> 1) & 1);
    tc::fence_after();
    const float inv = 1.f / lsum;
    bf16* dst = r < rows ? p.out + ((size_t)(q_base + it.q_tok0 + r / G) * p.n_q_heads + kvh * G + r % G) * kDh
                         : nullptr;
#pragma unroll
    for (int c0 = CPT * h; c0 < CPT * (h + 1); c0 += 32) {
      uint32_t o[32];
      tc::ld32x32(t_o + lane_base + c0, o);
      tc::wait_ld();
      if (dst) {
#pragma unroll
        for (int c = 0; c < 32; c += 8) {
          float f[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(o[c + e]) * inv;
          *reinterpret_cast<uint4*>(dst + c0 + c) = pack8(f);
        }
      }
    }
  }
}

// Persistent prefill role: warps 0..11 of the calling CTA pull tiles t from the
// atomic queue q (tiles are items[t / Hkv] x kv head t % Hkv, longest first),
// allocating TMEM on the first tile and re-arming the mbarriers per tile.
// bar: a named barrier id for the kThreads prefill threads. `done` (CTA count)
// resets the queue once every CTA of the launch has left it.
template <int kSW>
PPD_DEV void tile_queue(const CUtensorMap* kv_map, const AttnParams& p, uint8_t* smem, const AttnItem* items,
                        int n_tiles, int warp, int lane, int bar, int* q, int* done, int n_ctas, int* s_next) {
  const Smem S(smem);
  const int tid = warp * 32 + lane;
  bool first = true;
  for (;;) {
    if (tid == 0) *s_next = atomicAdd(q, 1);
    tc::fence_before();
    named_barrier_sync(bar, threads_for(kSW));  // previous tile retired; next index published
    tc::fence_after();
    const int t = *s_next;
    if (t >= n_tiles) break;
    if (first && warp == 2) tc::alloc(S.tmem_slot, kTmemCols);
    if (tid == 0) init_barriers<kSW>(S, !first);
    tc::fence_before();
    named_barrier_sync(bar, threads_for(kSW));
    tc::fence_after();
    first = false;
    const AttnItem it = items[t / p.n_kv_heads];
    tile<kSW>(kv_map, p, S, it, t % p.n_kv_heads, *S.tmem_slot, warp, lane, false);
  }
  if (!first && warp == 2) tc::dealloc(*S.tmem_slot, kTmemCols);
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(done, 1) == n_ctas - 1) {  // last CTA out resets the queue for the next launch
      *q = 0;
      *done = 0;
      __threadfence();
    }
  }
}

}  // namespace pftc
}  // namespace ppdk
