// common.cuh — shared device helpers for the sm_100a kernels of the PPD data path.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define PPD_DEV __device__ __forceinline__

// Host: true the first time it is called for the current device with this
// mask (function attributes such as the dynamic shared-memory limit belong to
// the function's per-device context, so a process driving several GPUs, e.g.
// the engine's disaggregated layouts, must set them on every device).
inline bool first_on_device(unsigned long long* mask) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return true;
  const unsigned long long bit = 1ull << dev;
  if (__atomic_fetch_or(mask, bit, __ATOMIC_ACQ_REL) & bit) return false;
  return true;
}

// Host: SM count of the current device (queried once per device; B200: 148).
// Grids, persistent-kernel slots and schedule cuts are sized from it.
inline int device_sms() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  int n = __atomic_load_n(&cache[dev], __ATOMIC_ACQUIRE);
  if (n > 0) return n;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  __atomic_store_n(&cache[dev], n, __ATOMIC_RELEASE);
  return n;
}

namespace ppdk {

typedef __nv_bfloat16 bf16;

PPD_DEV float bf2f(bf16 v) { return __bfloat162float(v); }
PPD_DEV bf16 f2bf(float v) { return __float2bfloat16_rn(v); }
PPD_DEV float rbf(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }

// 8 bf16 packed in a uint4 <-> 8 floats
PPD_DEV void unpack8(const uint4& v, float* f) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}
PPD_DEV uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
PPD_DEV uint4 pack8(const float* f) {
  return make_uint4(pack2(f[0], f[1]), pack2(f[2], f[3]), pack2(f[4], f[5]), pack2(f[6], f[7]));
}

PPD_DEV uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// Deterministic random-init value; identical to oracle/model_oracle.c
// mo_weight_bf16 (same hash, same exact fp32 arithmetic, RNE to bf16).
PPD_DEV bf16 weight_value(uint64_t seed, int tensor, int layer, uint64_t idx) {
  uint64_t key = seed * 0x9E3779B97F4A7C15ULL + ((uint64_t)tensor << 56) +
                 ((uint64_t)layer << 44) + idx;
  uint64_t z = mix64(key);
  float u = __fmul_rn((float)(uint32_t)(z >> 40), 0x1p-24f);
  float v = __fsub_rn(__fmul_rn(2.0f, u), 1.0f);
  float w = __fmul_rn(v, 0.034641016f);
  return __float2bfloat16_rn(w);
}

PPD_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
PPD_DEV float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ---- mbarrier / bulk-async copy (TMA 1-D) PTX wrappers -------------------
PPD_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
PPD_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
PPD_DEV void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
PPD_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
PPD_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
PPD_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
PPD_DEV bool mbar_try_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
PPD_DEV void mbar_wait(uint64_t* bar, uint32_t phase) {
  while (!mbar_try_wait(bar, phase)) {
  }
}
// L2 eviction policy for streams read exactly once per step (weights, cached
// K/V): their lines go first, so the step's small working set (K-split
// partials, activations, residual) stays L2-resident between producer and
// consumer kernels instead of being evicted by the 40 GB stream
PPD_DEV uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// global -> shared bulk copy, completion counted on an mbarrier (bytes % 16 == 0)
PPD_DEV void bulk_g2s(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// explicit shared-state-space accesses: shared buffers carved out of the
// dynamic smem go through generic pointers, for which the compiler emits
// generic LD.E / ST.E (slower than LDS / STS on the same smem)
PPD_DEV void sts_f32(const void* p, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(smem_u32(p)), "f"(v) : "memory");
}
PPD_DEV void sts_f32x2(const void* p, float a, float b) {
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(smem_u32(p)), "f"(a), "f"(b) : "memory");
}
PPD_DEV float lds_f32(const void* p) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
PPD_DEV void sts_u128(void* p, const uint4& v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(p)), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

PPD_DEV void named_barrier_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---- cp.async (Ampere-style) -----------------------------------------------
PPD_DEV void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
PPD_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
PPD_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

}  // namespace ppdk

namespace ppdk {
// ---- programmatic dependent launch (PDL) ----------------------------------
// pdl_wait: block until the preceding kernel in the stream has completed and
// its memory is visible (no-op when launched without the PDL attribute).
// pdl_trigger: allow the next kernel to start launching (its prologue and any
// weight prefetch overlap this kernel's tail).
PPD_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
PPD_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// Entry of a light (no shared memory, short) kernel. kEarly: let the next
// kernel launch BEFORE waiting on our predecessor, so a heavy successor (GEMM /
// attention) gets its CTAs resident as the heavy predecessor's CTAs retire and
// starts streaming its weights / cached K/V (inputs this kernel does not
// write) into that tail. Heavy kernels trigger only after their own wait, so
// at most heavy -> light -> heavy are in flight (no unbounded launch cascade).
template <bool kEarly>
PPD_DEV void pdl_enter() {
  if (kEarly) {
    pdl_trigger();
    pdl_wait();
  } else {
    pdl_wait();
    pdl_trigger();
  }
}
}  // namespace ppdk
