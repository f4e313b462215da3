// ops.cu — K6: small fused elementwise / reduction kernels of the forward step
// (embedding gather, residual-add + RMSNorm, RoPE + paged KV write, SiLU-mul,
// greedy argmax) and the deterministic random-init fills. All HBM-bound; one
// CTA per token row with 16-byte vector accesses. Rounding points follow
// oracle/model_oracle.c exactly (IEEE _rn intrinsics, no contraction).
#include "common.cuh"
#include "kernels.h"
#include "ops_dev.cuh"

#include <algorithm>
#include <cstdlib>

namespace ppdk {

namespace {
constexpr int kNormMaxThreads = 640;  // add_rmsnorm: at most 640 threads; one 8-element chunk each up to d = 4096
constexpr int kNormPre = 4;           // K-partial slices whose loads are issued together (decode: <= 4)

// sum over the CTA (any multiple of 32 threads up to 1024)
PPD_DEV float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  float r = 0.f;
  if (threadIdx.x < 32) {
    r = threadIdx.x < (int)(blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    r = warp_sum(r);
    if (threadIdx.x == 0) red[32] = r;
  }
  __syncthreads();
  r = red[32];
  __syncthreads();
  return r;
}
}  // namespace

// ------------------------------------------------------------------ fills
__global__ void fill_random_kernel(bf16* dst, uint64_t n, uint64_t seed, int tensor, int layer) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = weight_value(seed, tensor, layer, i);
}
cudaError_t launch_fill_random(bf16* dst, uint64_t n, uint64_t seed, int tensor, int layer,
                               cudaStream_t s) {
  fill_random_kernel<<<device_sms() * 8, 256, 0, s>>>(dst, n, seed, tensor, layer);
  return cudaGetLastError();
}

// weight matrix [N][K] (row-major): element (n, k) = counter hash of n*K + k
__global__ void fill_matrix_kernel(bf16* dst, uint64_t n, uint64_t seed, int tensor, int layer) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = weight_value(seed, tensor, layer, i);
}
cudaError_t launch_fill_matrix(bf16* dst, uint64_t N, uint64_t K, uint64_t seed, int tensor, int layer,
                               cudaStream_t s) {
  fill_matrix_kernel<<<device_sms() * 8, 256, 0, s>>>(dst, N * K, seed, tensor, layer);
  return cudaGetLastError();
}

__global__ void fill_qkv_kernel(bf16* dst, int qd, int kd, int d, uint64_t seed, int layer) {
  const uint64_t n = (uint64_t)(qd + 2 * kd) * d;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t r = i / d, c = i % d;
    int tensor;
    uint64_t lr;
    if (r < (uint64_t)qd) { tensor = 1; lr = r; }
    else if (r < (uint64_t)(qd + kd)) { tensor = 2; lr = r - qd; }
    else { tensor = 3; lr = r - qd - kd; }
    dst[i] = weight_value(seed, tensor, layer, lr * d + c);
  }
}
cudaError_t launch_fill_qkv(bf16* dst, int qd, int kd, int d, uint64_t seed, int layer, cudaStream_t s) {
  fill_qkv_kernel<<<device_sms() * 8, 256, 0, s>>>(dst, qd, kd, d, seed, layer);
  return cudaGetLastError();
}

__global__ void fill_bias_kernel(float* dst, int qd, int kd, uint64_t seed, int layer) {
  int n = qd + 2 * kd;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int tensor, lr;
    if (i < qd) { tensor = 9; lr = i; }
    else if (i < qd + kd) { tensor = 10; lr = i - qd; }
    else { tensor = 11; lr = i - qd - kd; }
    dst[i] = bf2f(weight_value(seed, tensor, layer, (uint64_t)lr));
  }
}
cudaError_t launch_fill_bias(float* dst, int qd, int kd, uint64_t seed, int layer, cudaStream_t s) {
  fill_bias_kernel<<<64, 256, 0, s>>>(dst, qd, kd, seed, layer);
  return cudaGetLastError();
}

__global__ void fill_gate_up_kernel(bf16* dst, int F, int d, uint64_t seed, int layer) {
  const uint64_t n = (uint64_t)2 * F * d;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t r = i / d, c = i % d;
    uint64_t grp = r / 128, within = r % 128;
    int tensor = within < 64 ? 5 : 6;  // gate | up
    uint64_t lr = grp * 64 + (within & 63);
    dst[i] = weight_value(seed, tensor, layer, lr * d + c);
  }
}
cudaError_t launch_fill_gate_up(bf16* dst, int F, int d, uint64_t seed, int layer, cudaStream_t s) {
  fill_gate_up_kernel<<<device_sms() * 8, 256, 0, s>>>(dst, F, d, seed, layer);
  return cudaGetLastError();
}

__global__ void fill_const_kernel(bf16* dst, uint64_t n, float v) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = f2bf(v);
}
cudaError_t launch_fill_const(bf16* dst, uint64_t n, float v, cudaStream_t s) {
  fill_const_kernel<<<device_sms(), 256, 0, s>>>(dst, n, v);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ embed
template <bool kEarly>
__global__ void embed_kernel(const int* tokens, const bf16* embed, bf16* x, int d) {
  pdl_enter<kEarly>();
  const int r = blockIdx.x;
  const uint4* src = reinterpret_cast<const uint4*>(embed + (size_t)tokens[r] * d);
  uint4* dst = reinterpret_cast<uint4*>(x + (size_t)r * d);
  for (int c = threadIdx.x; c < d / 8; c += blockDim.x) dst[c] = src[c];
}
cudaError_t launch_embed(const int* tokens, const bf16* embed, bf16* x, int T, int d, cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  return launch_pdl(pdl_overlap() ? embed_kernel<true> : embed_kernel<false>, dim3(T), dim3(128), 0, s, tokens,
                    embed, x, d);
}

// --------------------------------------------------- residual add + RMSNorm
// v = x (+ rbf(sum of delta partials) | + delta_bf16); x <- v ; out = rbf(rbf(v) * inv_rms) * w
// One CTA per row; thread t owns the 8-element chunks t, t + blockDim, ...
// (kCh of them: one at d <= 4096, so every chunk's loads are in flight at once).
template <bool kWriteX, bool kEarly, int kCh>
__global__ void __launch_bounds__(kCh == 1 ? 512 : kNormMaxThreads, kCh == 1 ? 2 : 1) add_rmsnorm_kernel(
    bf16* x, const float* df, GemmParts parts, const bf16* db, const bf16* w,
    bf16* out, const int* rows, int d, float eps) {
  __shared__ float red[33];
  pdl_enter<kEarly>();
  const size_t row = rows ? (size_t)rows[blockIdx.x] : (size_t)blockIdx.x;
  const int nc = d / 8;
  float v[kCh][8];
  float ss = 0.f;
  // every chunk's loads are issued before the first store of x (a store in
  // between would order the next chunk's loads behind it: x may alias df)
#pragma unroll
  for (int k = 0; k < kCh; ++k) {
    int c = threadIdx.x + k * blockDim.x;
    if (c < nc) {
      unpack8(reinterpret_cast<const uint4*>(x + row * d)[c], v[k]);
      if (df) {
        add_delta8<false, kNormPre>(v[k], df, parts.stride, parts.valid(c * 8, (int)row), row, d, c);
      } else if (db) {
        float dv[8];
        unpack8(reinterpret_cast<const uint4*>(db + row * d)[c], dv);
#pragma unroll
        for (int j = 0; j < 8; ++j) v[k][j] = rbf(__fadd_rn(v[k][j], dv[j]));
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) ss += v[k][j] * v[k][j];
    }
  }
  if (kWriteX && (df || db)) {
#pragma unroll
    for (int k = 0; k < kCh; ++k) {
      int c = threadIdx.x + k * blockDim.x;
      if (c < nc) reinterpret_cast<uint4*>(x + row * d)[c] = pack8(v[k]);
    }
  }
  ss = block_sum(ss, red);
  const float inv = rms_inv(ss, d, eps);
  const size_t orow = rows ? (size_t)blockIdx.x : row;
#pragma unroll
  for (int k = 0; k < kCh; ++k) {
    int c = threadIdx.x + k * blockDim.x;
    if (c < nc) reinterpret_cast<uint4*>(out + orow * d)[c] = norm8(v[k], inv, w, c);
  }
}

template <bool kWriteX>
cudaError_t launch_norm(int n_rows, bf16* x, const float* df, const GemmParts& parts, const bf16* db,
                        const bf16* w, bf16* out, const int* rows, int d, float eps, cudaStream_t s) {
  const int nc = d / 8;
  const int ch = nc <= 512 ? 1 : std::max(2, (nc + kNormMaxThreads - 1) / kNormMaxThreads);
  const int threads = ((nc + ch - 1) / ch + 31) / 32 * 32;
  const bool early = pdl_overlap();
#define PPD_NORM(CH)                                                                                      \
  if (ch <= CH)                                                                                           \
    return launch_pdl(early ? add_rmsnorm_kernel<kWriteX, true, CH> : add_rmsnorm_kernel<kWriteX, false, CH>, \
                      dim3(n_rows), dim3(threads), 0, s, x, df, parts, db, w, out, rows, d, eps);
  PPD_NORM(1)
  PPD_NORM(2)
  PPD_NORM(4)
#undef PPD_NORM
  return cudaErrorInvalidValue;  // d > 20480
}

cudaError_t launch_add_rmsnorm(bf16* x, const float* delta_f32, const GemmParts& parts, const bf16* delta_bf16,
                               const bf16* w, bf16* h, int T, int d, float eps, cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  return launch_norm<true>(T, x, delta_f32, parts, delta_bf16, w, h, nullptr, d, eps, s);
}

cudaError_t launch_final_norm(const bf16* x, const float* delta_f32, const GemmParts& parts,
                              const bf16* delta_bf16, const int* rows, int n_rows, const bf16* w,
                              bf16* out, int T, int d, float eps, cudaStream_t s) {
  if (n_rows == 0) return cudaSuccess;
  return launch_norm<false>(n_rows, const_cast<bf16*>(x), delta_f32, parts, delta_bf16, w, out, rows, d, eps, s);
}

// ------------------------------------------------------- RoPE + KV write
// One CTA per token row. Each thread owns 4 consecutive rotary pairs (i..i+3,
// i+64..i+67) of one q/k head, or 4 consecutive dims of one v head, and reads
// the fp32 GEMM output (all K-split partial slices) with 16-byte loads.
template <bool kEarly>
__global__ void rope_kv_kernel(RopeArgs a, int T) {
  pdl_enter<kEarly>();
  const int r = blockIdx.x;
  const int n = rope_units_per_row(a);
  for (int u = blockIdx.y * blockDim.x + threadIdx.x; u < n; u += gridDim.y * blockDim.x)
    rope_kv_unit<false, 4>(a, r, u, a.parts.valid(rope_unit_col(a, u), r));
}

cudaError_t launch_rope_kv_write(const float* qkv, const GemmParts& parts, const float* bias, const int* row_seq,
                                 const int* row_pos, const int* block_tables, int max_blocks,
                                 const float* rope_cos, const float* rope_sin, bf16* q_out,
                                 bf16* kv_pool, int T, int Hq, int Hkv, int Dh, int n_layers,
                                 int layer, int block_tokens, cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  const RopeArgs a{qkv,     parts, bias, row_seq, row_pos, block_tables, max_blocks, rope_cos, rope_sin,
                   q_out,   kv_pool, Hq,  Hkv,     Dh,      n_layers,     layer,      block_tokens};
  // (row, eighth of the row's rotary/v units): 8 CTAs per token row, one unit
  // per thread at the Llama-3-8B shape (896 units), for memory parallelism
  return launch_pdl(pdl_overlap() ? rope_kv_kernel<true> : rope_kv_kernel<false>, dim3(T, 8), dim3(128), 0, s, a, T);
}

// ------------------------------------------------------------- SiLU * up
// gate/up come interleaved in 64-column groups (launch_fill_gate_up layout);
// each thread produces 4 outputs from one float4 of gate and one of up.
// Each thread produces kSiluQ quads (256 * 4 columns apart) and issues all of
// their slice loads before the first store.
template <bool kEarly, int kSiluQ>
__global__ void silu_mul_kernel(const float* gu, GemmParts parts, bf16* m, int F) {
  pdl_enter<kEarly>();
  const int r = blockIdx.y;
  const int j0 = (blockIdx.x * blockDim.x * kSiluQ + threadIdx.x) * 4;
  float4 g[kSiluQ], u[kSiluQ];
#pragma unroll
  for (int q = 0; q < kSiluQ; ++q) {
    const int j = j0 + q * (int)blockDim.x * 4;
    if (j < F) silu4_load<false>(gu, parts.stride, parts.valid((j >> 6) * 128, r), F, r, j, g[q], u[q]);
  }
#pragma unroll
  for (int q = 0; q < kSiluQ; ++q) {
    const int j = j0 + q * (int)blockDim.x * 4;
    if (j < F) silu4_store(g[q], u[q], m, F, r, j);
  }
}
cudaError_t launch_silu_mul(const float* gu, const GemmParts& parts, bf16* m, int T, int F, cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  // small batches: one quad per thread, so the grid still covers the SMs
  // (T=16: 224 CTAs instead of 112)
  if (T < 64) {
    dim3 grid((F / 4 + 255) / 256, T);
    return launch_pdl(pdl_overlap() ? silu_mul_kernel<true, 1> : silu_mul_kernel<false, 1>, grid, dim3(256), 0, s, gu,
                      parts, m, F);
  }
  dim3 grid((F / 4 + 256 * 2 - 1) / (256 * 2), T);
  return launch_pdl(pdl_overlap() ? silu_mul_kernel<true, 2> : silu_mul_kernel<false, 2>, grid, dim3(256), 0, s, gu,
                    parts, m, F);
}

// ---------------------------------------------------------------- argmax
template <bool kEarly>
__global__ void argmax_kernel(const float* logits, int V, int* out) {
  pdl_enter<kEarly>();
  const float* row = logits + (size_t)blockIdx.x * V;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  auto take = [&](float x, int v) {
    if (x > best || (x == best && v < bi)) {
      best = x;
      bi = v;
    }
  };
  if ((V & 3) == 0) {
    // 16-byte loads, two in flight per thread; a thread's indices only grow,
    // so the strict '>' keeps the lowest index among its ties
    const float4* r4 = reinterpret_cast<const float4*>(row);
    const int n4 = V >> 2;
    int i = threadIdx.x;
    for (; i + (int)blockDim.x < n4; i += 2 * blockDim.x) {
      const float4 a = r4[i], b = r4[i + blockDim.x];
      take(a.x, 4 * i); take(a.y, 4 * i + 1); take(a.z, 4 * i + 2); take(a.w, 4 * i + 3);
      const int j = i + blockDim.x;
      take(b.x, 4 * j); take(b.y, 4 * j + 1); take(b.z, 4 * j + 2); take(b.w, 4 * j + 3);
    }
    for (; i < n4; i += blockDim.x) {
      const float4 a = r4[i];
      take(a.x, 4 * i); take(a.y, 4 * i + 1); take(a.z, 4 * i + 2); take(a.w, 4 * i + 3);
    }
  } else {
    for (int v = threadIdx.x; v < V; v += blockDim.x) take(row[v], v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    float ob = __shfl_xor_sync(0xffffffffu, best, o);
    int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
  }
  __shared__ float sb[32];
  __shared__ int si[32];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { sb[w] = best; si[w] = bi; }
  __syncthreads();
  if (w == 0) {
    int nw = blockDim.x >> 5;
    best = l < nw ? sb[l] : -INFINITY;
    bi = l < nw ? si[l] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      float ob = __shfl_xor_sync(0xffffffffu, best, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    if (l == 0) out[blockIdx.x] = bi;
  }
}
cudaError_t launch_argmax(const float* logits, int n, int V, int* out, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  return launch_pdl(pdl_overlap() ? argmax_kernel<true> : argmax_kernel<false>, dim3(n), dim3(1024), 0, s, logits, V, out);
}

__global__ void f32_to_bf16_kernel(const float* in, bf16* out, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = f2bf(in[i]);
}
cudaError_t launch_f32_to_bf16(const float* in, bf16* out, uint64_t n, cudaStream_t s) {
  f32_to_bf16_kernel<<<device_sms() * 4, 256, 0, s>>>(in, out, n);
  return cudaGetLastError();
}

}  // namespace ppdk

namespace ppdk {
static int g_pdl_overlap = 0;  // measured: 2.5% slower decode step (tools/ab_step.py)
int pdl_overlap() { return pdl_enabled() && g_pdl_overlap; }
void set_pdl_overlap(int on) { g_pdl_overlap = on; }
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PPD_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
}  // namespace ppdk
