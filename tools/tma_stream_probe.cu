// tma_stream_probe.cu — how fast can 148 SMs stream a decode GEMM's weights
// into shared memory through TMA, with no math? Three access patterns over
// the same 235 MB (the Llama-3-8B gate|up matrix, 28672 x 4096 bf16):
//   A  2-D tensor boxes of 128 rows x 64 bf16 (128 B per row, rows 8 KB
//      apart) over the row-major matrix: the GEMM's weight stream today
//   B  the same boxes over a tiled copy where each box is one contiguous
//      16 KB run (layout [row tile][k block][128][64])
//   C  1-D bulk copies (cp.async.bulk) of contiguous 16 KB runs
//   D  A + the decode GEMM's activation box per stage (208 token rows x 64,
//      26.6 KB, L2-resident: every CTA reads the same 200 x 4096 matrix)
//   E  A + half that activation box (104 rows: the CTA-pair share)
//   F  D + the tcgen05 MMAs of each stage (M=128 weight rows x N=208 tokens,
//      4 x K=16, fp32 accumulator in TMEM; the stage is released by
//      tcgen05.commit): the decode GEMM's main loop without its epilogue
//   G  F with N=104
//   H  F + the epilogue of one 128 x 208 fp32 accumulator at the end (4
//      warps: tcgen05.ld 32x32b + coalesced st.global, 104 KB per CTA): the
//      drain every decode GEMM launch pays once
//   I  H with the TMEM loads only (no stores)   J  H with the stores only (no TMEM loads)
//   K  H with the tile staged in shared memory (st.shared) and written by ONE
//      1-D TMA bulk store (cp.async.bulk.global.shared::cta) per CTA
//   L  H writing only the first 104 tokens (half the bytes)
//   M  H with streaming stores (st.global.cs)
// Each CTA streams a contiguous range of (row tile, k block) items through an
// S-stage mbarrier ring (one elected thread issues; a consumer thread releases
// each stage as soon as it lands). Prints GB/s per pattern and ring depth.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tsp tools/tma_stream_probe.cu -lcuda && /tmp/tsp
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../paper_2603_13358_b200/csrc/tc_common.cuh"

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));       \
      return 1;                                                               \
    }                                                                         \
  } while (0)

constexpr int kRows = 28672, kK = 4096, kBM = 128, kBK = 64, kBox = kBM * kBK * 2;
constexpr int kTiles = kRows / kBM, kKb = kK / kBK, kItems = kTiles * kKb;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(su32(b)), "r"(ph)
        : "memory");
}

template <int kMode>
__global__ void __launch_bounds__(192) stream_kernel(const __grid_constant__ CUtensorMap map, const uint8_t* lin,
                                                    int stages, unsigned long long* sink,
                                                    const __grid_constant__ CUtensorMap xmap, int xbytes,
                                                    float* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  const int sb = kBox + xbytes;  // stage bytes
  uint64_t* full = (uint64_t*)(smem + stages * sb);
  uint64_t* empty = full + stages;
  __shared__ uint64_t acc_done;
  __shared__ uint32_t tslot_s;
  uint32_t& tslot = tslot_s;
  if (kMode >= 5 && threadIdx.x >= 32 && threadIdx.x < 64) ppdk::tc::alloc(&tslot_s, 256);
  if (threadIdx.x == 0) {
    bar_init(&acc_done, 1);
    for (int i = 0; i < stages; ++i) {
      bar_init(&full[i], 1);
      bar_init(&empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  ppdk::tc::fence_before();
  __syncthreads();
  ppdk::tc::fence_after();
  const long long x0 = (long long)blockIdx.x * kItems / gridDim.x, x1 = (long long)(blockIdx.x + 1) * kItems / gridDim.x;
  const int n = (int)(x1 - x0);
  if (threadIdx.x == 0) {
    for (int i = 0; i < n; ++i) {
      const int s = i % stages;
      if (i >= stages) wait(&empty[s], ((i / stages) - 1) & 1);
      const long long item = x0 + i;
      const int tile = (int)(item / kKb), kb = (int)(item % kKb);
      expect_tx(&full[s], kBox + xbytes);
      if (kMode >= 3)  // the activation box of this k block (modes 3..6)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
            "[%4];" ::"r"(su32(smem + s * sb + kBox)),
            "l"((uint64_t)&xmap), "r"(kb * kBK), "r"(0), "r"(su32(&full[s]))
            : "memory");
      if (kMode == 0 || kMode >= 3) {  // row-major matrix, box (kb*64, tile*128)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
            "[%4];" ::"r"(su32(smem + s * sb)),
            "l"((uint64_t)&map), "r"(kb * kBK), "r"(tile * kBM), "r"(su32(&full[s]))
            : "memory");
      } else if (kMode == 1) {  // tiled copy viewed as [items*128][64]: box (0, item*128)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
            "[%4];" ::"r"(su32(smem + s * sb)),
            "l"((uint64_t)&map), "r"(0), "r"((int)(item * kBM)), "r"(su32(&full[s]))
            : "memory");
      } else {  // 1-D bulk copy of the item's contiguous 16 KB
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                su32(smem + s * sb)),
            "l"(lin + item * kBox), "r"(kBox), "r"(su32(&full[s]))
            : "memory");
      }
    }
  } else if (kMode >= 5) {
    // MMA issuer (warp 1): the decode GEMM's per-stage tcgen05 work
    if (threadIdx.x >= 32 && threadIdx.x < 64) {
      const uint32_t tmem = tslot;
      if (threadIdx.x == 32) {
        const int N = xbytes / 128;
        const uint32_t idesc = ppdk::tc::idesc_bf16(128, N, false);
        for (int i = 0; i < n; ++i) {
          const int s = i % stages;
          wait(&full[s], (i / stages) & 1);
          ppdk::tc::fence_after();
          const uint32_t sa = su32(smem + s * sb);
          const uint64_t da = ppdk::tc::desc_kmajor_sw128(sa), db = ppdk::tc::desc_kmajor_sw128(sa + kBox);
#pragma unroll
          for (int k = 0; k < 4; ++k) ppdk::tc::mma_bf16_ss(tmem, da + 2 * k, db + 2 * k, idesc, (i > 0) || (k > 0));
          ppdk::tc::commit(&empty[s]);
        }
        ppdk::tc::commit(&acc_done);  // all MMAs retired
      }
      __syncwarp();
    }
  }
  if (kMode >= 7 && threadIdx.x >= 64) {  // epilogue warps 2..5 (TMEM lane quarters 2,3,0,1)
    const int w = threadIdx.x >> 5, lq = w & 3, ln = threadIdx.x & 31;
    wait(&acc_done, 0);
    ppdk::tc::fence_after();
    const int N = xbytes / 128;
    const uint32_t tbase = tslot + ((uint32_t)(lq * 32) << 16);
    float* dst = out + (size_t)blockIdx.x * 128 * N + lq * 32 + ln;
    unsigned acc = 0;
    const int ntok = kMode == 11 ? 104 : 200;
    for (int c0 = 0; c0 < ntok; c0 += 32) {
      uint32_t r[32];
      if (kMode != 9) {
        ppdk::tc::ld32x32(tbase + (uint32_t)c0, r);
        ppdk::tc::wait_ld();
      } else {
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) r[jj] = jj + c0;
      }
      const int nj = min(32, 200 - c0);
      if (kMode == 10) {  // stage [token][row] in the (now idle) stage ring
        float* st = reinterpret_cast<float*>(smem) + lq * 32 + ln;
#pragma unroll
        for (int jj = 0; jj < 32; ++jj)
          if (jj < nj) {
            const uint32_t a = su32(st + (c0 + jj) * 128);
            asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(r[jj]) : "memory");
          }
      } else if (kMode == 8) {
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) acc += r[jj];
      } else if (kMode == 12) {
#pragma unroll
        for (int jj = 0; jj < 32; ++jj)
          if (jj < nj) __stcs(dst + (size_t)(c0 + jj) * 128, __uint_as_float(r[jj]));
      } else {
        const int nn = min(nj, ntok - c0);
#pragma unroll
        for (int jj = 0; jj < 32; ++jj)
          if (jj < nn) dst[(size_t)(c0 + jj) * 128] = __uint_as_float(r[jj]);
      }
    }
    if (acc == 0xFFFFFFFFu) *sink = acc;
    if (kMode == 10) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (threadIdx.x == 64) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                         out + (size_t)blockIdx.x * 128 * N),
                     "r"(su32(smem)), "r"(200 * 128 * 4)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      }
    }
  }
  if (kMode >= 5) {
    ppdk::tc::fence_before();
    __syncthreads();
    if (threadIdx.x >= 32 && threadIdx.x < 64) ppdk::tc::dealloc(tslot, 256);
  }
  if (kMode < 5 && threadIdx.x == 32) {
    unsigned long long acc = 0;
    for (int i = 0; i < n; ++i) {
      const int s = i % stages;
      wait(&full[s], (i / stages) & 1);
      acc += smem[s * sb + (i & 1023)];
      arrive(&empty[s]);
    }
    if (acc == 0xFFFFFFFFFFFFFFFFull) *sink = acc;
  }
}

static bool make_map(CUtensorMap* m, void* base, uint64_t rows, uint64_t cols, int box_rows = kBM) {
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return cuTensorMapEncodeTiled(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static float* g_out = nullptr;
template <int kMode>
static int run(const char* name, const CUtensorMap& map, const uint8_t* lin, int grid, int stages,
               unsigned long long* sink, const CUtensorMap& xmap, int xbytes) {
  const int smem = 1024 + stages * (kBox + xbytes) + 2 * stages * 8;
  CK(cudaFuncSetAttribute(stream_kernel<kMode>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) stream_kernel<kMode><<<grid, 192, smem>>>(map, lin, stages, sink, xmap, xbytes, g_out);
  CK(cudaDeviceSynchronize());
  const int iters = 10;
  cudaEventRecord(a);
  for (int i = 0; i < iters; ++i) stream_kernel<kMode><<<grid, 192, smem>>>(map, lin, stages, sink, xmap, xbytes, g_out);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = (double)kItems * kBox;
  printf("{\"pattern\": \"%s\", \"grid\": %d, \"stages\": %d, \"us\": %.2f, \"weight_GBps\": %.1f, "
         "\"l2_to_smem_GBps\": %.1f}\n",
         name, grid, stages, ms * 1e3 / iters, bytes / (ms * 1e-3 / iters) / 1e9,
         bytes * (kBox + xbytes) / kBox / (ms * 1e-3 / iters) / 1e9);
  return 0;
}

int main() {
  cuInit(0);
  const size_t bytes = (size_t)kRows * kK * 2;
  uint8_t *w = nullptr, *t = nullptr;
  unsigned long long* sink = nullptr;
  CK(cudaMalloc(&w, bytes));
  CK(cudaMalloc(&t, bytes));
  CK(cudaMalloc(&sink, 8));
  CK(cudaMalloc(&g_out, (size_t)148 * 128 * 208 * 4 * 2));
  CK(cudaMemset(w, 1, bytes));
  CK(cudaMemset(t, 1, bytes));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint8_t* x = nullptr;
  CK(cudaMalloc(&x, (size_t)200 * kK * 2));
  CK(cudaMemset(x, 1, (size_t)200 * kK * 2));
  CUtensorMap m_rm, m_tiled, m_x208, m_x104;
  if (!make_map(&m_rm, w, kRows, kK) || !make_map(&m_tiled, t, (uint64_t)kItems * kBM, kBK) ||
      !make_map(&m_x208, x, 200, kK, 208) || !make_map(&m_x104, x, 200, kK, 104)) {
    printf("tensor map failed\n");
    return 1;
  }
  for (int stages : {4, 8}) {
    const int grid = sms;
    if (run<0>("A_rowmajor_2d_box", m_rm, w, grid, stages, sink, m_x208, 0)) return 1;
    if (run<2>("C_tiled_1d_bulk", m_tiled, t, grid, stages, sink, m_x208, 0)) return 1;
  }
  for (int stages : {3, 5}) {
    if (run<3>("D_weights_plus_act208", m_rm, w, sms, stages, sink, m_x208, 208 * 128)) return 1;
    if (run<4>("E_weights_plus_act104", m_rm, w, sms, stages, sink, m_x104, 104 * 128)) return 1;
    if (run<5>("F_D_plus_mma_n208", m_rm, w, sms, stages, sink, m_x208, 208 * 128)) return 1;
    if (run<6>("G_E_plus_mma_n104", m_rm, w, sms, stages, sink, m_x104, 104 * 128)) return 1;
    if (run<7>("H_F_plus_final_epilogue", m_rm, w, sms, stages, sink, m_x208, 208 * 128)) return 1;
    if (run<8>("I_H_tmem_loads_only", m_rm, w, sms, stages, sink, m_x208, 208 * 128)) return 1;
    if (run<9>("J_H_stores_only", m_rm, w, sms, stages, sink, m_x208, 208 * 128)) return 1;
    if (run<10>("K_H_smem_staged_tma_bulk_store", m_rm, w, sms, stages, sink, m_x208, 208 * 128)) return 1;
    if (run<11>("L_H_half_bytes", m_rm, w, sms, stages, sink, m_x208, 208 * 128)) return 1;
    if (run<12>("M_H_streaming_stores", m_rm, w, sms, stages, sink, m_x208, 208 * 128)) return 1;
  }
  return 0;
}
