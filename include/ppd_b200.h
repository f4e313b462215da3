/* ppd_b200.h — the C-ABI between the host C++ PPD engine and the sm_100a device
 * path (libppd_b200.so). Plain pointers and sizes; no torch types; no exception
 * crosses it. Every entry returns an int status (PPD_OK == 0); on failure
 * ppd_last_error() returns a thread-local message.
 *
 * The reference (/root/reference/proj) has no FFI: its execute path is four
 * analytic cost functions called from the simulator's event handlers
 * (SURVEY.md §8b). Each entry below names the reference interface it replaces:
 *
 *   ppd_prefill(FULL)    replaces cost::full_prefill_time     costmodel.hpp:85, costmodel.cpp:318-322
 *                        (called simulator.cpp:327)
 *   ppd_prefill(APPEND)  replaces cost::append_prefill_time   costmodel.hpp:86, costmodel.cpp:324-331
 *                        (called simulator.cpp:328-329)
 *   ppd_step             replaces cost::decode_step_time x interference_multiplier
 *                        costmodel.hpp:97-100, costmodel.cpp:347-379 (called simulator.cpp:397):
 *                        one fused iteration = decode rows + an optional append/prefill chunk
 *   ppd_kv_copy          replaces cost::kv_transfer_time      costmodel.hpp:88-91, costmodel.cpp:333-345
 *                        (called simulator.cpp:354)
 *   ppd_kv_pool_init     replaces Node::prefix_cache           simulator.cpp:125 (token counts only)
 *                        with a paged HBM pool; block tables stay host-side
 *
 * Errors the reference reports with std::invalid_argument (costmodel.cpp:319,
 * :325-327, :335, :374-375) return PPD_ERR_INVALID with the same condition text.
 */
#ifndef PPD_B200_H
#define PPD_B200_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define PPD_OK 0
#define PPD_ERR_INVALID (-1) /* invalid argument (reference: std::invalid_argument) */
#define PPD_ERR_CUDA (-2)    /* CUDA / driver failure */
#define PPD_ERR_OOM (-3)     /* device memory exhausted */
#define PPD_ERR_STATE (-4)   /* call out of order (e.g. step before weights/pool) */

#define PPD_PREFILL_FULL 0   /* cost::PrefillKind::full   (costmodel.hpp:12) */
#define PPD_PREFILL_APPEND 1 /* cost::PrefillKind::append */

typedef struct ppd_model_cfg {
  int32_t n_layers, d_model, n_q_heads, n_kv_heads, head_dim, d_ff, vocab;
  float rms_eps, rope_theta;
  int32_t qkv_bias; /* Qwen2.5: 1 */
} ppd_model_cfg;

typedef struct ppd_dev ppd_dev; /* one GPU worker: weights, KV pool, streams */

const char* ppd_last_error(void);
int ppd_version(void);
int ppd_device_count(int32_t* n);

/* max_step_tokens: largest sum(q_len) of one ppd_step; max_step_seqs: largest n_seqs. */
int ppd_dev_open(int32_t gpu, const ppd_model_cfg* cfg, int32_t max_step_tokens,
                 int32_t max_step_seqs, ppd_dev** out);
int ppd_dev_close(ppd_dev* dev);
int ppd_load_random_weights(ppd_dev* dev, uint64_t seed);
int ppd_kv_pool_init(ppd_dev* dev, int32_t block_tokens, int32_t num_blocks);
/* bytes of one KV block (all layers, K and V, all kv heads) */
int ppd_kv_block_bytes(const ppd_model_cfg* cfg, int32_t block_tokens, uint64_t* bytes);
int ppd_kv_pool_ptr(ppd_dev* dev, void** ptr, uint64_t* bytes);
/* Synchronous host <-> pool copies of a byte range (after the device's queued
 * work): KV snapshot / restore, and how tests seed a cached context. */
int ppd_kv_pool_write(ppd_dev* dev, uint64_t offset, const void* host, uint64_t bytes);
int ppd_kv_pool_read(ppd_dev* dev, uint64_t offset, void* host, uint64_t bytes);

/* One fused iteration over n_seqs sequences. Sequence s contributes q_len[s]
 * new tokens at positions ctx[s] .. ctx[s]+q_len[s]-1; their K/V are written
 * into the pool through its block table row, then every new token attends to
 * positions 0..its own (causal). q_len[s] == 1 is a decode row. For every s
 * with want_token[s] != 0 (all s when want_token is NULL) the greedy next
 * token after its last new token is written to out_tokens[s]. All arrays are
 * HOST arrays; the call copies them in, runs, and copies the tokens out. */
typedef struct ppd_batch {
  int32_t n_seqs;
  const int32_t* q_len;        /* [n_seqs] */
  const int32_t* ctx;          /* [n_seqs] */
  const int32_t* tokens;       /* [sum q_len] */
  const int32_t* block_tables; /* [n_seqs * max_blocks] */
  int32_t max_blocks;
  const int32_t* want_token;   /* [n_seqs] or NULL */
} ppd_batch;

/* Synchronous: returns when out_tokens is filled. *out_ms (may be NULL) is the
 * device time of the step (CUDA events on the compute stream). */
int ppd_step(ppd_dev* dev, const ppd_batch* batch, int32_t* out_tokens, float* out_ms);
/* Asynchronous pair: submit enqueues H2D + kernels + D2H into pinned staging. */
int ppd_step_submit(ppd_dev* dev, const ppd_batch* batch);
int ppd_step_wait(ppd_dev* dev, int32_t* out_tokens, float* out_ms);
/* fp32 logits of the last step's want_token rows, [n_seqs][vocab] (host). */
int ppd_last_logits(ppd_dev* dev, float* out, int64_t max_floats);

/* Prefill seam. FULL: n_ctx must be 0 and tokens holds the whole history
 * (the P node's full recompute, simulator.cpp:309-311). APPEND: tokens holds
 * the n_new new tokens, attending n_ctx cached ones (simulator.cpp:282-289). */
int ppd_prefill(ppd_dev* dev, int32_t kind, const int32_t* tokens, int32_t n_new, int32_t n_ctx,
                const int32_t* block_table, int32_t n_blocks, int32_t* out_token, float* out_ms);

/* Token-granular KV transfer of positions [start, start+n_tokens) of one
 * sequence from src's pool to dst's pool (the P->D hop, simulator.cpp:349-356).
 * The copy kernel runs on dst's transfer stream and pulls over peer pointers
 * (NVLink when src/dst are different GPUs), fenced after src's last submitted
 * step. Bytes moved = n_tokens * kv bytes/token.
 *
 * ppd_kv_copy_submit is asynchronous: no host synchronisation, no allocation
 * on the hot path (block tables travel through a preallocated pinned/device
 * ring), and dst's compute stream is NOT blocked, so the hop overlaps dst's
 * decode steps. Rows that read the copied tokens may be stepped only after
 * ppd_kv_copy_wait(dst, ticket) returned (tickets of one dst are waited for
 * in submission order, from any one thread; at most 64 in flight per dst).
 * *out_ms: device time of the copy (CUDA events on the transfer stream).
 * ppd_kv_copy = submit + wait (it first retires older tickets of dst). */
int ppd_kv_copy_submit(ppd_dev* src, ppd_dev* dst, const int32_t* src_block_table,
                       const int32_t* dst_block_table, int32_t n_blocks, int32_t start,
                       int32_t n_tokens, uint64_t* ticket);
int ppd_kv_copy_wait(ppd_dev* dst, uint64_t ticket, float* out_ms);
int ppd_kv_copy(ppd_dev* src, ppd_dev* dst, const int32_t* src_block_table,
                const int32_t* dst_block_table, int32_t n_blocks, int32_t start,
                int32_t n_tokens, float* out_ms);
/* NVLink roofline probe: GB/s of `bytes` moved src_gpu -> dst_gpu, best of
 * `iters` (mode 0 copy engines / cudaMemcpyPeerAsync, mode 1 SM pull kernel
 * on dst, the K7 access pattern). src_gpu == dst_gpu measures an HBM copy. */
int ppd_p2p_bandwidth(int32_t src_gpu, int32_t dst_gpu, uint64_t bytes, int32_t iters, int32_t mode,
                      double* gbs);
/* Weights of one node: bytes resident and how many open devices share them
 * (nodes on the same GPU with the same shape and seed share one copy). */
int ppd_weights_info(ppd_dev* dev, uint64_t* bytes, int32_t* shared_by);

/* ---- instrumentation (CUDA events on the compute stream, per kernel class) ----
 * With profiling on, every attention launch and every GEMM of a step is
 * bracketed by CUDA events; ppd_step_wait accumulates the durations. The
 * counters count launches of this library's own kernels vs library GEMMs. */
typedef struct ppd_dev_stats {
  int64_t steps;
  int64_t own_launches;   /* kernels compiled in libppd_b200.so */
  int64_t lib_launches;   /* vendor-library launches (cuBLAS GEMM calls) */
  int64_t attn_launches;
  double attn_ms, gemm_ms;   /* only with profiling on */
  double attn_bytes;         /* algorithmic bytes of all attention launches */
  double step_ms;            /* device time of all steps */
} ppd_dev_stats;
int ppd_dev_set_profiling(ppd_dev* dev, int32_t on);
int ppd_dev_get_stats(ppd_dev* dev, ppd_dev_stats* out);
int ppd_dev_reset_stats(ppd_dev* dev);

/* ---- kernel-level entry points (device pointers; used by parity tests) ----
 * stream: cudaStream_t or NULL for the legacy default stream. The GEMM ops are
 * asynchronous on that stream; the others synchronise before returning. */
/* attention over a paged pool (num_blocks blocks) for one layer, through the
 * same work-item builder and kernel as ppd_step. q [total_q][Hq][Dh] bf16
 * (roped, device), out same shape bf16 (device). q_start [n_seqs+1], ctx
 * [n_seqs], block_tables [n_seqs*max_blocks] are HOST int32. Synchronous. */
int ppd_op_attention(const ppd_model_cfg* cfg, const void* q, const void* kv_pool,
                     int32_t num_blocks, int32_t block_tokens, int32_t layer, int32_t n_seqs,
                     const int32_t* q_start, const int32_t* ctx, const int32_t* block_tables,
                     int32_t max_blocks, void* out, void* stream);
/* C[M][N] = A[M][K] . B[N][K]^T ; bf16 in, out_f32 ? fp32 : bf16 out.
 * ppd_op_gemm: the cuBLAS library GEMM (the reference the kernel is tested against);
 * ppd_op_gemm_tc: the tcgen05/TMEM kernel used by ppd_step; with splits > 1 it
 * writes `splits` fp32 K-partial slices of M*N floats (their sum is C). */
int ppd_op_gemm(const void* A, const void* B, void* C, int32_t M, int32_t N, int32_t K,
                int32_t out_f32, void* stream);
int ppd_op_gemm_tc(const void* A, const void* B, void* C, int32_t M, int32_t N, int32_t K,
                   int32_t out_f32, int32_t splits, void* stream);
/* The MLP up-projection with SiLU fused into the tcgen05 epilogue:
 * m[M][N/2] = bf16(silu(g) * u), g/u the fp32 products of the interleaved
 * gate|up weight B [N][K] (64-row groups: rows [128j, 128j+64) gate rows
 * [64j, 64j+64), rows [128j+64, 128j+128) the matching up rows). N % 128 == 0.
 * Asynchronous on `stream`. */
int ppd_op_gemm_silu(const void* A, const void* B, void* m, int32_t M, int32_t N, int32_t K,
                     void* stream);
/* The forward step's fp32 GEMM path: C = sum of K-partial slices C + j*stride.
 * Uniform split (kbt == 0): all n slices valid. Balanced partition: slot c owns
 * items [c*total/slots, (c+1)*total/slots) of the (tile, k-block) space, tile
 * t = (col / rows) * n_tiles_t + tok / bn; slices j < owner(t*kbt+kbt-1) -
 * owner(t*kbt) + 1 are valid, owner(x) = ceil((x+1)*slots/total) - 1.
 * C must hold max_slices * M * N floats. Asynchronous on `stream`. */
typedef struct ppd_gemm_parts {
  int32_t n, kbt, slots, rows, bn, n_tiles_t;
  int64_t total;
  uint64_t stride;
  int32_t dp; /* leading whole-K (data-parallel) tiles; the stream-K ranges cover the rest */
} ppd_gemm_parts;
int ppd_op_gemm_parts(const void* A, const void* B, void* C, int32_t M, int32_t N, int32_t K,
                      int32_t max_slices, ppd_gemm_parts* parts, void* stream);
/* process-wide kernel tuning knobs (tests and sweeps; defaults are tuned):
 *   "gemm_pair"   -1 auto (CTA-pair tcgen05 kernel for >= 48 token rows),
 *                  0 single-CTA kernel, 1 CTA-pair kernel for every shape
 *   "gemm_stages"  cap on the GEMM smem ring depth (0 = as many as fit)
 *   "gemm_sched"  -1 auto, 0 uniform K split, 1 balanced partition (fp32 path)
 *   "mlp_fused"    1 gate|up GEMM with the SiLU epilogue, 0 (default) fp32
 *                  partials + a separate SiLU kernel
 *   "gemm_multi_sub" 1 (default): 257..512 token rows run as one unit of two
 *                  token sub-tiles per weight stage for the wide projections
 *                  and for narrow ones whose CTA-pair tiles fill the SMs in one
 *                  round; 2: every projection; 3: wide ones only; 0: separate
 *                  token tiles
 *   "gemm_epi_pipe" 1 (default): the plain GEMM epilogue keeps the next
 *                  32-column TMEM load in flight while it stores the current
 *                  chunk; 0: load, wait, store per chunk
 *   "l2_hint"      3 (default): TMA loads of streams read once per step carry
 *                  an L2 evict-first policy -- bit 0 the GEMM weights (steps
 *                  whose token rows fit one unit), bit 1 the decode K/V;
 *                  0: no cache hint
 *   "gemm_occ2"    0 (default) off, -1 auto (<= 128 token rows), 1 on: two co-resident
 *                  CTAs per SM with half-depth rings
 *   "attn_fused"   1 (default): a mixed decode + prefill step runs its
 *                  attention as ONE launch (K2) when its prefill tiles fit
 *                  under the decode rows' K/V streaming, else the decode
 *                  kernel then the persistent prefill queue; 2: K2 for every
 *                  mixed step; 0: never K2
 *   "attn_pf_ctas" K2 prefill CTA count (0 = cost model, default)
 *   "attn_pf_persist" 1 (default): pure prefill steps run a persistent
 *                  tcgen05 kernel over an atomic tile queue; 0: one CTA per tile
 *   "layer_kernel" 0 (default): per-op kernels; 1: steps of <= 256 token
 *                  rows on a GPU driven by one device handle run each layer
 *                  after attention as ONE persistent launch (o, add+norm,
 *                  gate|up, SiLU, down, add+norm, next qkv, RoPE/KV write)
 *   "layer_l2_ahead" K8 weight k-blocks prefetched into L2 beyond the ring
 *   "layer_stages" K8 smem ring depth cap (0 = as deep as fits)
 * Unknown names -> PPD_ERR_INVALID. Every change makes devices re-capture
 * their step graphs with the newly selected kernels. */
int ppd_set_tuning(const char* name, int32_t value);
/* deterministic random-init fill, identical to the oracle's mo_weight_bf16 */
int ppd_op_fill_random(void* dst, uint64_t n, uint64_t seed, int32_t tensor, int32_t layer,
                       void* stream);

#ifdef __cplusplus
}
#endif
#endif
