// kv_copy.cu — K7: token-granular paged-KV transfer between two pools (the
// P->D hop that replaces cost::kv_transfer_time, reference costmodel.cpp:333-345,
// called at simulator.cpp:354 with need = ctx + new - have tokens).
//
// The sequence positions are identical on both sides, so for every 16-token
// block b touched by [start, start+n) and every (layer, K|V, kv head) the bytes
// to move are one contiguous run of (tokens in b) x head_dim x 2 B in both
// pools. One warp moves one run with 16-byte vector accesses; when the pools
// live on different GPUs the source is a peer (NVLink) pointer and the copy is a
// pull by the destination GPU.
#include "common.cuh"
#include "kernels.h"

namespace ppdk {

__global__ void kv_copy_kernel(KvCopyParams p) {
  const int lane = threadIdx.x & 31;
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int n_warps = (gridDim.x * blockDim.x) >> 5;
  const int BT = p.block_tokens;
  const int first_b = p.start / BT;
  const int last_b = (p.start + p.n_tokens - 1) / BT;
  const int per_block = p.n_layers * 2 * p.n_kv_heads;
  const long units = (long)(last_b - first_b + 1) * per_block;
  const size_t row_bytes = (size_t)p.head_dim * 2;
  for (long u = warp_global; u < units; u += n_warps) {
    int bi = (int)(u / per_block);
    int rest = (int)(u % per_block);  // (layer, kv, head) flattened = slice index inside a block
    int b = first_b + bi;
    int t0 = max(p.start, b * BT) - b * BT;
    int t1 = min(p.start + p.n_tokens, (b + 1) * BT) - b * BT;
    size_t slice = (size_t)rest * BT;  // rows of head_dim within the block
    const uint8_t* src = reinterpret_cast<const uint8_t*>(p.src_pool) +
                         (((size_t)p.src_blocks[b] * per_block * BT) + slice + t0) * row_bytes;
    uint8_t* dst = reinterpret_cast<uint8_t*>(p.dst_pool) +
                   (((size_t)p.dst_blocks[b] * per_block * BT) + slice + t0) * row_bytes;
    const int n16 = (int)((t1 - t0) * row_bytes / 16);
    const uint4* __restrict__ s4 = reinterpret_cast<const uint4*>(src);
    uint4* __restrict__ d4 = reinterpret_cast<uint4*>(dst);
    int i = lane;
    // a whole 16-token run (4 KB at head_dim 128) is 8 x 512 B: issue all loads first
    for (; i + 7 * 32 < n16; i += 8 * 32) {
      uint4 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = __ldcs(s4 + i + k * 32);
#pragma unroll
      for (int k = 0; k < 8; ++k) __stcs(d4 + i + k * 32, v[k]);
    }
    for (; i < n16; i += 32) __stcs(d4 + i, __ldcs(s4 + i));
  }
}

cudaError_t launch_kv_copy(const KvCopyParams& p, cudaStream_t s) {
  if (p.n_tokens <= 0) return cudaSuccess;
  const int BT = p.block_tokens;
  long units = (long)((p.start + p.n_tokens - 1) / BT - p.start / BT + 1) * p.n_layers * 2 * p.n_kv_heads;
  const long cap = (long)device_sms() * 64;
  long warps = units < cap ? units : cap;
  int blocks = (int)((warps + 7) / 8);
  kv_copy_kernel<<<blocks, 256, 0, s>>>(p);
  return cudaGetLastError();
}

// Peer-bandwidth probe: a flat pull of n16 16-byte words (src may be a peer
// pointer), the same access pattern as kv_copy_kernel's runs.
__global__ void pull_copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, long n16) {
  const long stride = (long)gridDim.x * blockDim.x;
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n16; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldcs(src + i + k * stride);
#pragma unroll
    for (int k = 0; k < 8; ++k) __stcs(dst + i + k * stride, v[k]);
  }
  for (; i < n16; i += stride) __stcs(dst + i, __ldcs(src + i));
}

cudaError_t launch_pull_copy(const uint4* src, uint4* dst, long n16, cudaStream_t s) {
  pull_copy_kernel<<<device_sms() * 8, 256, 0, s>>>(src, dst, n16);
  return cudaGetLastError();
}

}  // namespace ppdk
