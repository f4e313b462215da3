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

PPD_DEV void tma_load_2d(void* smem, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
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

}  // namespace

// Persistent: grid = min(units, 148); CTA c processes units c, c + grid, ...
// where a unit is (weight tile, token tile, K split), weight-tile-major so the
// CTAs running concurrently share weight tiles and token tiles through L2. The
// producer streams stages across unit boundaries without draining; the MMA
// warp alternates between two TMEM accumulators (when 2*BN <= 512 columns) so
// the epilogue of unit i overlaps the MMAs of unit i+1.
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x,
                   GemmTcParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = p.stages;
  const int x_bytes = p.bn * kBK * 2;
  const int stage_bytes = kWBytes + x_bytes;  // both multiples of 1 KB
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);
  uint64_t* empty = full + S;
  uint64_t* acc_full = empty + S;   // [2]
  uint64_t* acc_empty = acc_full + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tiles_w = (p.N + kBM - 1) / kBM;
  const int n_tiles_t = (p.T + p.bn - 1) / p.bn;
  const int n_units = n_tiles_w * n_tiles_t * p.splits;
  const int kb_total = (p.K + kBK - 1) / kBK;
  const int kb_per = (kb_total + p.splits - 1) / p.splits;
  const int n_acc = p.tmem_cols >= 2 * p.bn_cols ? 2 : 1;

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 4);  // one arrive per epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(p.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_trigger();  // the next kernel may launch; it waits for our completion itself

  // unit -> (weight tile, token tile, split); token tile fastest
  auto decode_unit = [&](int u, int& tw, int& tt, int& sp) {
    sp = u % p.splits;
    const int rest = u / p.splits;
    tt = rest % n_tiles_t;
    tw = rest / n_tiles_t;
  };

  if (warp == 0) {
    if (lane == 0) {
      // Weights do not depend on the previous kernel: stream the first stages of
      // W before waiting on it (PDL), then the activations.
      int npre = 0;
      if ((int)blockIdx.x < n_units) {
        int tw, tt, sp;
        decode_unit(blockIdx.x, tw, tt, sp);
        const int kb0 = sp * kb_per, kb1 = min(kb_total, kb0 + kb_per);
        npre = min(S, max(0, kb1 - kb0));
        for (int i = 0; i < npre; ++i) {
          mbar_arrive_expect_tx(&full[i], stage_bytes);
          tma_load_2d(smem + i * stage_bytes, &map_w, (kb0 + i) * kBK, tw * kBM, &full[i]);
        }
      }
      pdl_wait();
      int it = 0;  // global stage counter across units
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        int tw, tt, sp;
        decode_unit(u, tw, tt, sp);
        const int kb0 = sp * kb_per, kb1 = min(kb_total, kb0 + kb_per);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % S;
          uint8_t* sw = smem + s * stage_bytes;
          if (it >= npre) {
            if (it >= S) mbar_wait(&empty[s], ((it / S) - 1) & 1);
            mbar_arrive_expect_tx(&full[s], stage_bytes);
            tma_load_2d(sw, &map_w, kb * kBK, tw * kBM, &full[s]);
          }
          tma_load_2d(sw + kWBytes, &map_x, kb * kBK, tt * p.bn, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(p.bn >> 3) << 17) |
                             ((uint32_t)(kBM >> 4) << 24);
      int it = 0, j = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++j) {
        int tw, tt, sp;
        decode_unit(u, tw, tt, sp);
        const int kb0 = sp * kb_per, kb1 = min(kb_total, kb0 + kb_per);
        const int acc = j % n_acc;
        const int use = j / n_acc;  // how many times this accumulator was used before
        if (use > 0) mbar_wait(&acc_empty[acc], (use - 1) & 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * p.bn_cols);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % S;
          mbar_wait(&full[s], (it / S) & 1);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + s * stage_bytes);
          const uint64_t da = sw128_kmajor_desc(sa);
          const uint64_t db = sw128_kmajor_desc(sa + kWBytes);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)  // 32 B per UMMA_K step inside the swizzle atom
            mma_bf16(d_tmem, da + (uint64_t)(k * 2), db + (uint64_t)(k * 2), idesc, (kb != kb0) || (k != 0));
          mma_commit(&empty[s]);  // smem slot free once these MMAs retire
        }
        mma_commit(&acc_full[acc]);
      }
    }
  } else if (warp >= 4) {
    pdl_wait();  // outputs are written only after the predecessor retired
    const int q = warp & 3;  // TMEM lane quarter owned by this warp
    int j = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++j) {
      int tw, tt, sp;
      decode_unit(u, tw, tt, sp);
      const int acc = j % n_acc;
      const int use = j / n_acc;
      const int row = tw * kBM + q * 32 + lane;
      const int t0 = tt * p.bn;
      mbar_wait(&acc_full[acc], use & 1);
      tc_fence_after();
      float* out32 = reinterpret_cast<float*>(p.out) + (size_t)sp * p.split_stride;
      __nv_bfloat16* out16 = reinterpret_cast<__nv_bfloat16*>(p.out);
      const uint32_t t_acc = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * p.bn_cols);
      const int ncols = min(p.bn, p.T - t0);
      for (int c0 = 0; c0 < ncols; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(t_acc + (uint32_t)c0, r);
        if (row < p.N) {
          const int nj = min(32, ncols - c0);
          if (p.out_f32) {
            float* dst = out32 + (size_t)(t0 + c0) * p.ldo + row;
#pragma unroll
            for (int jj = 0; jj < 32; ++jj)
              if (jj < nj) dst[(size_t)jj * p.ldo] = __uint_as_float(r[jj]);
          } else {
            __nv_bfloat16* dst = out16 + (size_t)(t0 + c0) * p.ldo + row;
#pragma unroll
            for (int jj = 0; jj < 32; ++jj)
              if (jj < nj) dst[(size_t)jj * p.ldo] = __float2bfloat16_rn(__uint_as_float(r[jj]));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
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

int gemm_tc_plan_splits(int T, int N, int K) {
  const int bn = T >= kMaxBN ? kMaxBN : ((T + 15) / 16) * 16;
  const int tiles = ((N + kBM - 1) / kBM) * ((T + bn - 1) / bn);
  const int kb = (K + kBK - 1) / kBK;
  // Persistent CTAs take units round-robin, so the step costs
  //   rounds(s) x (bytes of one unit) = ceil(tiles*s/148) x (W slab / s + fp32 partial write + read).
  // Pick the split count minimising it (s <= 8, >= 4 K-blocks per split).
  const double w_unit = double(kBM) * K * 2.0;
  const double out_unit = double(bn) * kBM * 4.0 * 2.0;
  int best = 1;
  double best_cost = 1e300;
  // the callers' fp32 workspaces hold 8 x 256 token rows of partial slices
  for (int s = 1; s <= 8 && kb / s >= 4 && s * T <= 8 * 256; ++s) {
    const int rounds = (tiles * s + 147) / 148;
    const double cost = rounds * (w_unit / s + (s > 1 ? out_unit : out_unit * 0.5));
    if (cost < best_cost * 0.97) {  // prefer fewer partial slices unless clearly better
      best_cost = cost;
      best = s;
    }
  }
  return best;
}

cudaError_t gemm_tc_run(const bf16* X, const bf16* W, void* out, int T, int N, int K, bool out_f32, int splits,
                        size_t split_stride, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  if (K % 8 != 0) return cudaErrorInvalidValue;  // TMA row stride must be 16 B aligned
  const int bn = T >= kMaxBN ? kMaxBN : ((T + 15) / 16) * 16;
  if (splits < 1) splits = 1;
  if (splits > 1 && !out_f32) return cudaErrorInvalidValue;
  GemmTcParams p{};
  p.out = out;
  p.T = T;
  p.N = N;
  p.K = K;
  p.ldo = N;
  p.bn = bn;
  p.out_f32 = out_f32 ? 1 : 0;
  p.splits = splits;
  p.split_stride = split_stride ? split_stride : (size_t)T * N;
  // accumulator columns per unit (power of two >= bn); two accumulators when they fit
  p.bn_cols = bn <= 32 ? 32 : bn <= 64 ? 64 : bn <= 128 ? 128 : 256;
  p.tmem_cols = 2 * p.bn_cols <= 512 ? 2 * p.bn_cols : p.bn_cols;
  const int stage_bytes = kWBytes + bn * kBK * 2;
  int stages = kSmemBudget / stage_bytes;
  stages = stages > kMaxStages ? kMaxStages : stages;
  static const int stage_cap = [] {
    const char* e = std::getenv("PPD_GEMM_STAGES");
    return e ? std::atoi(e) : 0;
  }();
  if (stage_cap > 0 && stage_cap < stages) stages = stage_cap;
  p.stages = stages;
  const int smem = 1024 + stages * stage_bytes + 256;
  CUtensorMap mw, mx;
  if (!get_map(&mw, W, N, K, kBM) || !get_map(&mx, X, T, K, bn)) return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 1024 + kSmemBudget + 256);
    attr = true;
  }
  const int units = ((N + kBM - 1) / kBM) * ((T + bn - 1) / bn) * splits;
  const int grid = units < 148 ? units : 148;
  return launch_pdl(gemm_tc_kernel, dim3(grid), dim3(kThreads), (size_t)smem, s, mw, mx, p);
}

}  // namespace ppdk
