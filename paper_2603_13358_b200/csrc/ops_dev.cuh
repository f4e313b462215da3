// ops_dev.cuh — per-element formulas of the small fused ops (K6), shared by
// the stand-alone kernels in ops.cu and the glue phases of the decode layer
// kernel (layer_tc.cu), so both paths round at the same points as
// oracle/model_oracle.c (IEEE _rn intrinsics, no contraction).
//
// kCg: read the fp32 GEMM partial slices with ld.global.cg (L2 only). The
// layer kernel reads slices written by other SMs earlier in the same launch,
// so it must not hit stale L1 lines; stand-alone kernels read through L1.
#pragma once
#include "common.cuh"
#include "gemm_tc.h"
#include "kernels.h"

namespace ppdk {

template <bool kCg>
PPD_DEV float4 ld_f4(const float* p) {
  if (kCg) return __ldcg(reinterpret_cast<const float4*>(p));
  return *reinterpret_cast<const float4*>(p);
}
template <bool kCg>
PPD_DEV uint4 ld_u4(const void* p) {
  if (kCg) return __ldcg(reinterpret_cast<const uint4*>(p));
  return *reinterpret_cast<const uint4*>(p);
}

PPD_DEV float4 add4(float4 a, const float4& v) {
  a.x = __fadd_rn(a.x, v.x);
  a.y = __fadd_rn(a.y, v.y);
  a.z = __fadd_rn(a.z, v.z);
  a.w = __fadd_rn(a.w, v.w);
  return a;
}

// 0 + slice 0 + slice 1 + ... (fp32, slice order) of n >= 1 partial slices of
// 4 floats. The loads of the first min(n, kPre) slices are issued before the
// first add (one L2 round trip for them instead of one each); the decode
// layer kernel's glue runs at 8 warps per SM and is latency-bound otherwise.
constexpr int kMaxSlices = 8;
template <bool kCg, int kPre = 2>
PPD_DEV float4 sum_slices4(const float* p, size_t stride, int n) {
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
  float4 v[kPre];
#pragma unroll
  for (int i = 0; i < kPre; ++i)
    if (i < n) v[i] = ld_f4<kCg>(p + i * stride);
#pragma unroll
  for (int i = 0; i < kPre; ++i)
    if (i < n) a = add4(a, v[i]);
  for (int pp = kPre; pp < n; ++pp) a = add4(a, ld_f4<kCg>(p + pp * stride));
  return a;
}

// n valid K-partial slices of 4 consecutive output columns (+ bias), slice order
template <bool kRound, bool kCg, int kPre = 2>
PPD_DEV float4 ld_sum4(const float* base, size_t stride, int n, const float* bias, int col) {
  float4 a = sum_slices4<kCg, kPre>(base + col, stride, n);
  if (bias) a = add4(a, *reinterpret_cast<const float4*>(bias + col));
  if (!kRound) return a;
  return make_float4(rbf(a.x), rbf(a.y), rbf(a.z), rbf(a.w));
}

PPD_DEV void st_bf16x4(bf16* dst, float a, float b, float c, float d) {
  *reinterpret_cast<uint2*>(dst) = make_uint2(pack2(a, b), pack2(c, d));
}

// residual add of one 8-element chunk c of `row`: v = rbf(x + rbf(sum of its n delta slices))
template <bool kCg, int kPre = 2>
PPD_DEV void add_delta8(float* v, const float* df, size_t stride, int n, size_t row, int d, int c) {
  const float* base = df + row * d + (size_t)c * 8;
  const float4 a = sum_slices4<kCg, kPre>(base, stride, n);
  const float4 b = sum_slices4<kCg, kPre>(base + 4, stride, n);
  const float acc[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = rbf(__fadd_rn(v[j], rbf(acc[j])));
}

// RMSNorm output chunk: o = rbf(rbf(v * inv) * w)
PPD_DEV uint4 norm8(const float* v, float inv, const bf16* w, int c) {
  float wv[8], o[8];
  unpack8(reinterpret_cast<const uint4*>(w)[c], wv);
#pragma unroll
  for (int j = 0; j < 8; ++j) o[j] = __fmul_rn(rbf(__fmul_rn(v[j], inv)), wv[j]);
  return pack8(o);
}
PPD_DEV float rms_inv(float ss, int d, float eps) {
  return __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(ss, (float)d), eps)));
}

// SiLU(gate) * up for 4 outputs m[r][j..j+4) from the interleaved gate|up
// partials (64-column groups, launch_fill_gate_up). Fast exp/div: within
// 2 ulp of the oracle's fp32, rounded to bf16 next.
// (gate and up of one output share a 128-column weight tile: one slice count n)
// the two halves of silu4: gather gate / up sums, then compute + store, so a
// caller can issue several units' loads before the first store
template <bool kCg>
PPD_DEV void silu4_load(const float* gu, size_t stride, int n, int F, int r, int j, float4& g, float4& u) {
  const float* row = gu + (size_t)r * 2 * F;
  const int grp = j >> 6, within = j & 63;
  g = ld_sum4<false, kCg>(row, stride, n, nullptr, grp * 128 + within);
  u = ld_sum4<false, kCg>(row, stride, n, nullptr, grp * 128 + 64 + within);
}
PPD_DEV void silu4_store(const float4& g, const float4& u, bf16* m, int F, int r, int j) {
  const float gv[4] = {g.x, g.y, g.z, g.w}, uv[4] = {u.x, u.y, u.z, u.w};
  float o[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) o[e] = __fmul_rn(__fdividef(gv[e], __fadd_rn(1.0f, __expf(-gv[e]))), uv[e]);
  st_bf16x4(m + (size_t)r * F + j, o[0], o[1], o[2], o[3]);
}
template <bool kCg>
PPD_DEV void silu4(const float* gu, size_t stride, int n, bf16* m, int F, int r, int j) {
  float4 g, u;
  silu4_load<kCg>(gu, stride, n, F, r, j, g, u);
  silu4_store(g, u, m, F, r, j);
}

PPD_DEV int rope_units_per_row(const RopeArgs& a) { return (a.Hq + a.Hkv) * (a.Dh / 8) + a.Hkv * a.Dh / 4; }

// qkv output column of unit u's first element (its 128-column weight tile = one head)
PPD_DEV int rope_unit_col(const RopeArgs& a, int u) {
  const int per_head = a.Dh / 8, n_rot = (a.Hq + a.Hkv) * per_head;
  if (u < n_rot) return (u / per_head) * a.Dh + (u % per_head) * 4;
  return (a.Hq + a.Hkv) * a.Dh + (u - n_rot) * 4;
}
// unit u of row r: 4 rotary pairs (i..i+3, i+64..i+67) of one q/k head, or 4
// dims of one v head; n = valid qkv slices of the unit's head
template <bool kCg, int kPre = 2>
PPD_DEV void rope_kv_unit(const RopeArgs& a, int r, int u, int n) {
  const int half = a.Dh / 2;
  const int qd = a.Hq * a.Dh, kd = a.Hkv * a.Dh, W = qd + 2 * kd;
  const int pos = a.row_pos[r], seq = a.row_seq[r];
  const int blk = a.block_tables[(size_t)seq * a.max_blocks + pos / a.block_tokens];
  const int tok = pos % a.block_tokens;
  const float* row = a.qkv + (size_t)r * W;
  const int per_head = half / 4;  // rotary units per head
  const int n_rot = (a.Hq + a.Hkv) * per_head;
  if (u < n_rot) {
    const float* cs = a.rope_cos + (size_t)pos * half;
    const float* sn = a.rope_sin + (size_t)pos * half;
    const int head = u / per_head, i = (u % per_head) * 4;
    const int col = head * a.Dh + i;  // k heads follow q heads in the fused layout
    const float4 x1 = ld_sum4<true, kCg, kPre>(row, a.parts.stride, n, a.bias, col);
    const float4 x2 = ld_sum4<true, kCg, kPre>(row, a.parts.stride, n, a.bias, col + half);
    const float4 c = *reinterpret_cast<const float4*>(cs + i);
    const float4 sv = *reinterpret_cast<const float4*>(sn + i);
    const float a0 = rbf(__fsub_rn(__fmul_rn(x1.x, c.x), __fmul_rn(x2.x, sv.x)));
    const float a1 = rbf(__fsub_rn(__fmul_rn(x1.y, c.y), __fmul_rn(x2.y, sv.y)));
    const float a2 = rbf(__fsub_rn(__fmul_rn(x1.z, c.z), __fmul_rn(x2.z, sv.z)));
    const float a3 = rbf(__fsub_rn(__fmul_rn(x1.w, c.w), __fmul_rn(x2.w, sv.w)));
    const float b0 = rbf(__fadd_rn(__fmul_rn(x2.x, c.x), __fmul_rn(x1.x, sv.x)));
    const float b1 = rbf(__fadd_rn(__fmul_rn(x2.y, c.y), __fmul_rn(x1.y, sv.y)));
    const float b2 = rbf(__fadd_rn(__fmul_rn(x2.z, c.z), __fmul_rn(x1.z, sv.z)));
    const float b3 = rbf(__fadd_rn(__fmul_rn(x2.w, c.w), __fmul_rn(x1.w, sv.w)));
    bf16* dst;
    if (head < a.Hq) {
      dst = a.q_out + ((size_t)r * a.Hq + head) * a.Dh;
    } else {
      dst = a.kv + ((((size_t)blk * a.n_layers + a.layer) * 2 + 0) * a.Hkv + (head - a.Hq)) * a.block_tokens * a.Dh +
            (size_t)tok * a.Dh;
    }
    st_bf16x4(dst + i, a0, a1, a2, a3);
    st_bf16x4(dst + i + half, b0, b1, b2, b3);
  } else {
    const int v = (u - n_rot) * 4;
    const int hk = v / a.Dh, dd = v % a.Dh;
    const float4 x = ld_sum4<true, kCg, kPre>(row, a.parts.stride, n, a.bias, qd + kd + v);
    bf16* dst = a.kv + ((((size_t)blk * a.n_layers + a.layer) * 2 + 1) * a.Hkv + hk) * a.block_tokens * a.Dh +
                (size_t)tok * a.Dh + dd;
    st_bf16x4(dst, x.x, x.y, x.z, x.w);
  }
}

}  // namespace ppdk
