// device.cu — the C-ABI device worker (include/ppd_b200.h): weights resident in
// HBM, the paged KV pool, per-step metadata staging, and the fused forward step
// that replaces the reference's analytic service times (costmodel.cpp:318-379).
//
// One ppd_step = one iteration of a node's engine loop: every sequence in the
// batch contributes q_len new tokens (1 for a decode row, m for an append /
// prefill chunk). All rows go through the same projection GEMMs, so an append
// chunk rides inside the decode step (the paper's PPD argument);
// attention for decode rows and prefill tiles is ONE launch (attention.cu).
#include <cublas_v2.h>
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <atomic>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "../../include/ppd_b200.h"
#include "gemm.h"
#include "gemm_tc.h"
#include "common.cuh"
#include "kernels.h"

using namespace ppdk;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CU(expr)                                                                         \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess)                                                               \
      return fail(_e == cudaErrorMemoryAllocation ? PPD_ERR_OOM : PPD_ERR_CUDA,          \
                  std::string(#expr) + ": " + cudaGetErrorString(_e));                   \
  } while (0)

#define CHECK_ARG(cond, msg) \
  do {                       \
    if (!(cond)) return fail(PPD_ERR_INVALID, msg); \
  } while (0)

constexpr int kMaxRope = 1 << 17;  // positions covered by the RoPE table

// process-wide tuning (ppd_set_tuning); each change bumps the epoch so devices
// re-capture their step graphs with the newly selected kernels
int g_tuning_epoch = 0;
// gate|up GEMM with the SiLU epilogue writing bf16 m directly (else fp32
// partials + silu_mul_kernel). 0 never, 1 always, 2 (default) for steps of at
// least kMlpFusedMinRows token rows. Decode-size steps: no gain (within 1%,
// tools/ab_step.py, 48 steps per arm; the K-split partition balances better).
// Prefill-size steps: 8-16% faster steps (tools/ab_knobs.sh: the fp32 gate|up
// round trip is 2 x T x 28672 x 4 B per layer, 0.94 GB at T = 4096).
int g_mlp_fused = 2;
// workspaces sized for two K-partial slices of a max-size step (see alloc_workspaces)
bool g_ws_two_slices = true;
constexpr int kMlpFusedMinRows = 512;
// K8 decode layer kernel (layer_tc.cu) for steps of <= 256 token rows: tuning
// "layer_kernel" (0 default = the per-op kernels, 1 = K8). Measured slower
// than the per-op path at B = 16 / 64 / 200 (+24-45%, tools/ab_step.py,
// tools/k8_trace.py), so it is an option, not the default.
bool g_layer_kernel = false;
int g_layer_l2_ahead = 16;  // tuning "layer_l2_ahead"
int g_layer_stages = 0;     // tuning "layer_stages": ring depth cap (0 = as deep as fits)
// ppd_devs open per GPU: the layer kernel's grid barrier needs every SM of the
// GPU for its own CTAs, so it runs only on a GPU driven by ONE node (two
// nodes' layer kernels launched concurrently could each hold part of the SMs
// and wait on each other forever)
std::atomic<int> g_open_on_gpu[64];

struct Layer {
  bf16 *wqkv, *wo, *wgu, *wdown;
  float* bqkv;
};

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

int validate_cfg(const ppd_model_cfg* c) {
  CHECK_ARG(c, "null model cfg");
  CHECK_ARG(c->n_layers > 0 && c->d_model > 0 && c->n_q_heads > 0 && c->n_kv_heads > 0 &&
                c->d_ff > 0 && c->vocab > 0,
            "model cfg: sizes must be > 0");
  CHECK_ARG(c->head_dim == 128, "model cfg: head_dim must be 128 (sm_100a kernels)");
  CHECK_ARG(c->n_q_heads % c->n_kv_heads == 0, "model cfg: n_q_heads % n_kv_heads != 0");
  CHECK_ARG(c->n_q_heads / c->n_kv_heads <= 16, "model cfg: GQA group > 16");
  CHECK_ARG(c->d_model % 8 == 0 && c->d_model <= 8192, "model cfg: d_model % 8 or > 8192");
  CHECK_ARG(c->d_ff % 64 == 0, "model cfg: d_ff must be a multiple of 64");
  return PPD_OK;
}

}  // namespace

// One in-flight P->D KV hop on the destination's transfer stream
// (ppd_kv_copy_submit / ppd_kv_copy_wait): its timing events and the
// preallocated block-table staging (pinned host + device), reused per ticket.
struct CopySlot {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  int32_t* h_bt = nullptr;  // pinned [2 * cap]
  int32_t* d_bt = nullptr;  // device [2 * cap]
  int cap = 0;              // blocks per table
};
constexpr int kCopySlots = 64;

// Weights are read-only and a pure function of (shape, seed): nodes opened on
// the same GPU with the same model share one resident copy (an 8-node layout
// colocated on one B200 holds 16 GB of Llama-3-8B weights, not 128 GB).
struct SharedWeights {
  int gpu = 0;
  ppd_model_cfg cfg{};
  uint64_t seed = 0;
  void* mem = nullptr;
  size_t bytes = 0;
  int refs = 0;
};

struct ppd_dev {
  int gpu = 0;
  ppd_model_cfg cfg{};
  int max_T = 0, max_S = 0;
  size_t ws_rows = 0;  // token rows of fp32 GEMM-output workspace (holds K-partial slices)
  cudaStream_t compute = nullptr, xfer = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, compute_done = nullptr;
  // weights (possibly shared with other nodes on this GPU)
  SharedWeights* wshared = nullptr;
  bf16 *embed = nullptr, *lm_head = nullptr, *ones = nullptr;
  std::vector<Layer> layers;
  bool weights_ready = false;
  float *rope_cos = nullptr, *rope_sin = nullptr;
  // KV pool
  bf16* kv = nullptr;
  int bt = 0, nblocks = 0;
  uint64_t kv_bytes = 0;
  alignas(128) uint8_t kv_map[128];
  // activations / workspaces
  bf16 *x = nullptr, *h = nullptr, *q = nullptr, *attn = nullptr, *m = nullptr, *hl = nullptr;
  float *qkv32 = nullptr, *proj32 = nullptr, *gu32 = nullptr, *down32 = nullptr, *logits = nullptr;
  unsigned* layer_sync = nullptr;  // K8 grid-barrier counters [n_layers][8], zeroed per step
  float *ws_o = nullptr, *ws_ml = nullptr;
  int* counters = nullptr;
  int ws_slots = 0;
  // staging (pinned host + device)
  uint8_t* h_meta = nullptr;
  uint8_t* d_meta = nullptr;
  size_t meta_cap = 0;
  int* h_tokens_out = nullptr;
  int* d_tokens_out = nullptr;
  int pending = 0;  // sequences of the in-flight step (0 = none)
  int last_logit_rows = 0;
  // CUDA graphs of the forward pass, keyed by the step's shape (the metadata
  // contents change per step; the pointers and launch parameters do not)
  using GraphKey = std::tuple<int, int, int, int, int, long long, int>;
  std::map<GraphKey, cudaGraphExec_t> graphs;
  std::map<GraphKey, int> shape_seen;
  bool use_graphs = true;
  int tuning_epoch = 0;  // ppd_set_tuning generation the cached graphs were captured under
  // instrumentation
  bool profiling = false;
  ppd_dev_stats stats{};
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, int>> prof_marks;  // (kind 0 attn / 1 gemm, first event index)
  int ev_used = 0;
  // KV hops INTO this device (it is the destination): ticket t uses slot t % kCopySlots
  CopySlot copy[kCopySlots];
  std::atomic<uint64_t> copy_head{0}, copy_done{0};
  uint64_t peer_mask = 0;  // source GPUs peer access was enabled for
};

namespace {

// ------------------------------------------------------------ metadata
struct StepLayout {
  int n, T, maxb, n_out, n_items, n_ws, n_dec, n_cta;
  int n_pf;  // K2: prefill CTAs of the one-launch mixed attention (0 = not a mixed step)
  size_t off_seg;
  double attn_bytes;  // algorithmic bytes of one attention launch (one layer)
  size_t off_qstart, off_ctx, off_tokens, off_bt, off_rowseq, off_rowpos, off_outrows, off_items,
      total;
};

// Builds the attention work list for the batch. Decode rows (q_len == 1) get
// KV splits when the grid would otherwise under-fill the 148 SMs.
bool attention_tc_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PPD_ATTN_TC");
    return !(e && std::strcmp(e, "0") == 0);
  }();
  return on;
}

// Decode items come first, then prefill tiles (n_dec = number of decode items):
// decode rows run on paged_attention_kernel, prefill tiles of 128/G tokens on
// the tcgen05 kernel (or 64/G-token tiles on paged_attention_kernel when the
// tensor-core path is disabled).
void build_items(int n, const int32_t* q_len, const int32_t* ctx, int n_kv_heads, int group,
                 std::vector<AttnItem>& items, int& n_ws, int& n_dec) {
  items.clear();
  n_ws = 0;
  const int tq = std::max(1, (attention_tc_enabled() ? 128 : 64) / group);
  long base_ctas = 0;
  int n_decode = 0;
  for (int s = 0; s < n; ++s) {
    if (q_len[s] == 1) {
      ++n_decode;
      base_ctas += n_kv_heads;
    } else if (q_len[s] > 1) {
      base_ctas += (long)((q_len[s] + tq - 1) / tq) * n_kv_heads;
    }
  }
  int want = 1;
  const long target_ctas = 4L * device_sms();
  if (n_decode > 0 && base_ctas < target_ctas)
    want = (int)((target_ctas + base_ctas - 1) / std::max<long>(base_ctas, 1));
  for (int s = 0; s < n; ++s) {
    if (q_len[s] <= 0) continue;
    if (q_len[s] == 1) {
      int keys = ctx[s] + 1;
      int splits = std::min(want, (keys + 255) / 256);
      splits = std::max(splits, 1);
      int chunk = ((keys + splits - 1) / splits + 63) / 64 * 64;
      splits = (keys + chunk - 1) / chunk;
      for (int sp = 0; sp < splits; ++sp) {
        AttnItem it{};
        it.kind = 0;
        it.seq = s;
        it.q_tok0 = 0;
        it.n_q = 1;
        it.key_begin = sp * chunk;
        it.key_end = std::min(keys, (sp + 1) * chunk);
        it.split = sp;
        it.n_splits = splits;
        it.ws_index = splits > 1 ? n_ws + sp : -1;
        items.push_back(it);
      }
      if (splits > 1) n_ws += splits;
    } else {
      for (int t0 = 0; t0 < q_len[s]; t0 += tq) {
        AttnItem it{};
        it.kind = 1;
        it.seq = s;
        it.q_tok0 = t0;
        it.n_q = std::min(tq, q_len[s] - t0);
        it.n_splits = 1;
        it.ws_index = -1;
        items.push_back(it);
      }
    }
  }
  std::stable_partition(items.begin(), items.end(), [](const AttnItem& it) { return it.kind == 0; });
  n_dec = 0;
  for (const AttnItem& it : items) n_dec += it.kind == 0;
}

bool decode_persistent_enabled(int group) {
  static const bool on = [] {
    const char* e = std::getenv("PPD_DEC_PERSIST");
    return !(e && std::strcmp(e, "0") == 0);
  }();
  return on && group <= 5;
}

// Balanced decode schedule (decode_attention_kernel): the 64-key stages of all
// (decode sequence, kv head) pairs are cut into n_cta equal contiguous ranges;
// a pair cut by a range boundary becomes several key segments merged through
// the split workspace. Replaces the decode items of `items` (kept first) and
// fills seg_start[n_cta + 1].
void balance_decode(int n, const int32_t* q_len, const int32_t* ctx, int n_kv_heads, std::vector<AttnItem>& items,
                    int& n_ws, int& n_dec, std::vector<int>& seg_start, int kMaxCtas) {
  constexpr int kStageKeys = 64;
  long U = 0;
  for (int s = 0; s < n; ++s)
    if (q_len[s] == 1) U += (long)((ctx[s] + 1 + kStageKeys - 1) / kStageKeys) * n_kv_heads;
  std::vector<AttnItem> rest(items.begin() + n_dec, items.end());
  items.clear();
  seg_start.clear();
  n_ws = 0;
  if (U > 0) {
    long n_cta = std::min<long>(kMaxCtas, U);
    const long quota = (U + n_cta - 1) / n_cta;
    n_cta = (U + quota - 1) / quota;
    long u = 0;
    for (int s = 0; s < n; ++s) {
      if (q_len[s] != 1) continue;
      const int keys = ctx[s] + 1;
      const int nst = (keys + kStageKeys - 1) / kStageKeys;
      for (int h = 0; h < n_kv_heads; ++h) {
        std::vector<std::pair<int, int>> segs;
        for (int st = 0; st < nst;) {
          const long cta = u / quota;
          const int take = (int)std::min<long>(nst - st, (cta + 1) * quota - u);
          segs.push_back({st, st + take});
          st += take;
          u += take;
        }
        const int nseg = (int)segs.size();
        for (int k = 0; k < nseg; ++k) {
          AttnItem it{};
          it.kind = 0;
          it.seq = s;
          it.n_q = 1;
          it.key_begin = segs[k].first * kStageKeys;
          it.key_end = std::min(keys, segs[k].second * kStageKeys);
          it.split = k;
          it.n_splits = nseg;
          it.ws_index = nseg > 1 ? n_ws + k : -1;
          it.pad[0] = h;
          items.push_back(it);
        }
        if (nseg > 1) n_ws += nseg;
      }
    }
    // CTA c owns the segments whose first unit falls in [c*quota, (c+1)*quota)
    seg_start.assign(n_cta + 1, (int)items.size());
    long unit = 0;
    int c_next = 0;
    for (int i = 0; i < (int)items.size(); ++i) {
      const long cta = unit / quota;
      while (c_next <= cta) seg_start[c_next++] = i;
      unit += (items[i].key_end - items[i].key_begin + kStageKeys - 1) / kStageKeys;
    }
    while (c_next <= n_cta) seg_start[c_next++] = (int)items.size();
  }
  n_dec = (int)items.size();
  items.insert(items.end(), rest.begin(), rest.end());
}

// K2 (mixed_attention_kernel) SM split: n_pf CTAs start on the prefill queue,
// the decode schedule is cut for the other sms - n_pf SMs (two instances
// each) and those join the prefill queue when their decode work is done.
// Cost model (B200, tools/ab_step.py PPD_AB_MIX sweeps of attn_pf_ctas):
// decode streams min(5.6 TB/s, 44 GB/s per SM); a tile inside this launch
// costs ~4 us + 6 us per 128-key block on one SM; prefill work left at the
// end of decode is shared by all SMs.
int plan_mixed_split(double dec_bytes, const std::vector<double>& tile_cost, int sms) {
  const int n_tiles = (int)tile_cost.size();
  if (dec_bytes <= 0 || n_tiles == 0) return 0;
  double pf = 0;
  for (double c : tile_cost) pf += c;
  int best = 1;
  double best_t = 1e30;
  for (int n_pf = 1; n_pf <= std::min(n_tiles, sms - 2); ++n_pf) {
    const double t_dec = dec_bytes / std::min(5.6e12, (sms - n_pf) * 44e9);
    const double rest = std::max(0.0, pf - n_pf * t_dec);
    const double t = t_dec + rest / sms + (rest > 0 ? tile_cost[0] : 0.0);  // + one tile of tail
    if (t < best_t * 0.999) {
      best_t = t;
      best = n_pf;
    }
  }
  return best;
}

// tuning "attn_fused": 1 (default) K2 one-launch mixed attention when the
// prefill fits under the decode (mixed_step_fits_k2), 2 K2 for every mixed
// step (A/B), 0 never
int g_attn_fused = 1;

// K2 pays when the step's prefill tiles fit under its decode rows' K/V
// streaming (the decode-append mix of a large decode batch: B=200 + a
// 128-token append 12.7 vs 13.4 ms); when the prefill dominates (a turn-2+
// append of 1536 tokens beside a handful of decode rows, the PPD D node at
// low load) the persistent tcgen05 prefill kernel on all SMs after the
// decode kernel is faster (B=9 + 1536 over 2048: 31 vs 40 ms per step).
// Estimates: decode at 5.6 TB/s; prefill causal FLOPs at 0.7 PFLOP/s.
bool mixed_step_fits_k2(int n, const int32_t* q_len, const int32_t* ctx, int n_kv_heads, int G,
                        const std::vector<AttnItem>& items, int n_dec) {
  double dec_bytes = 0, pf_flop = 0;
  for (int s = 0; s < n; ++s)
    if (q_len[s] == 1) dec_bytes += (double)(ctx[s] + 1) * n_kv_heads * 2 * 128 * 2;
  for (size_t i = n_dec; i < items.size(); ++i) {
    const AttnItem& it = items[i];
    pf_flop += 4.0 * it.n_q * G * (ctx[it.seq] + it.q_tok0 + it.n_q) * 128.0 * n_kv_heads;
  }
  return pf_flop / 0.7e15 <= dec_bytes / 5.6e12;
}
int g_attn_pf_ctas = 0;          // tuning "attn_pf_ctas": force the K2 prefill CTA count (0 = cost model)
bool g_attn_pf_persist = true;  // tuning "attn_pf_persist": persistent tile queue for pure prefill steps

// The attention work of one step: decode items (balanced schedule), prefill
// tiles (longest first) and, for a mixed step, the K2 SM split n_pf.
void plan_attention(int n, const int32_t* q_len, const int32_t* ctx, int n_kv_heads, int G,
                    std::vector<AttnItem>& items, int& n_ws, int& n_dec, std::vector<int>& seg_start, int& n_pf) {
  build_items(n, q_len, ctx, n_kv_heads, G, items, n_ws, n_dec);
  const int sms = device_sms();
  seg_start.clear();
  n_pf = 0;
  if (!decode_persistent_enabled(G)) return;
  if (attention_tc_enabled() && g_attn_pf_persist && n_dec == 0 && !items.empty()) {
    // pure prefill step: longest tiles first for the persistent tile queue
    std::stable_sort(items.begin(), items.end(), [&](const AttnItem& a, const AttnItem& b) {
      return ctx[a.seq] + a.q_tok0 + a.n_q > ctx[b.seq] + b.q_tok0 + b.n_q;
    });
  }
  if (attention_tc_enabled() && n_dec > 0 && (int)items.size() > n_dec) {
    // longest prefill tiles first: the tile queues (K2 and the persistent
    // prefill kernel) hand them out in this order
    std::stable_sort(items.begin() + n_dec, items.end(), [&](const AttnItem& a, const AttnItem& b) {
      return ctx[a.seq] + a.q_tok0 + a.n_q > ctx[b.seq] + b.q_tok0 + b.n_q;
    });
  }
  if (attention_tc_enabled() && g_attn_fused && n_dec > 0 && (int)items.size() > n_dec &&
      (g_attn_fused == 2 || mixed_step_fits_k2(n, q_len, ctx, n_kv_heads, G, items, n_dec))) {
    std::vector<double> cost;
    for (size_t i = n_dec; i < items.size(); ++i) {
      const AttnItem& it = items[i];
      const double blocks = (ctx[it.seq] + it.q_tok0 + it.n_q + 127) / 128;
      for (int h = 0; h < n_kv_heads; ++h) cost.push_back(4.0e-6 + 6.0e-6 * blocks);
    }
    double dec_bytes = 0;
    for (int s = 0; s < n; ++s)
      if (q_len[s] == 1) dec_bytes += (double)(ctx[s] + 1) * n_kv_heads * 2 * 128 * 2;
    n_pf = g_attn_pf_ctas > 0 ? std::min<int>(g_attn_pf_ctas, (int)cost.size()) : plan_mixed_split(dec_bytes, cost, sms);
  }
  balance_decode(n, q_len, ctx, n_kv_heads, items, n_ws, n_dec, seg_start, n_pf > 0 ? 2 * (sms - n_pf) : 2 * sms);
  if (seg_start.empty()) n_pf = 0;
}

void clear_graphs(ppd_dev* d) {
  for (auto& kv : d->graphs) cudaGraphExecDestroy(kv.second);
  d->graphs.clear();
}

int ensure_meta(ppd_dev* d, size_t bytes) {
  if (bytes <= d->meta_cap) return PPD_OK;
  size_t cap = align_up(bytes * 2, 1 << 20);
  if (d->h_meta) cudaFreeHost(d->h_meta);
  if (d->d_meta) cudaFree(d->d_meta);
  d->h_meta = nullptr;
  d->d_meta = nullptr;
  CU(cudaMallocHost(&d->h_meta, cap));
  CU(cudaMalloc(&d->d_meta, cap));
  d->meta_cap = cap;
  clear_graphs(d);
  return PPD_OK;
}

int ensure_ws(ppd_dev* d, int slots) {
  if (slots <= d->ws_slots) return PPD_OK;
  int cap = std::max(slots, 1024);
  const int G = d->cfg.n_q_heads / d->cfg.n_kv_heads;
  if (d->ws_o) cudaFree(d->ws_o);
  if (d->ws_ml) cudaFree(d->ws_ml);
  d->ws_o = nullptr;
  d->ws_ml = nullptr;
  CU(cudaMalloc(&d->ws_o, (size_t)cap * d->cfg.n_kv_heads * G * 128 * sizeof(float)));
  CU(cudaMalloc(&d->ws_ml, (size_t)cap * d->cfg.n_kv_heads * G * 2 * sizeof(float)));
  d->ws_slots = cap;
  clear_graphs(d);
  return PPD_OK;
}

template <typename T>
T* at(uint8_t* base, size_t off) {
  return reinterpret_cast<T*>(base + off);
}

// Packs the batch into the pinned staging buffer (one H2D copy per step).
int pack_batch(ppd_dev* d, const ppd_batch* b, StepLayout& L, std::vector<AttnItem>& items) {
  CHECK_ARG(b && b->n_seqs > 0, "batch: n_seqs must be >= 1");
  CHECK_ARG(b->n_seqs <= d->max_S, "batch: n_seqs exceeds max_step_seqs");
  CHECK_ARG(b->q_len && b->ctx && b->tokens && b->block_tables, "batch: null array");
  CHECK_ARG(b->max_blocks > 0, "batch: max_blocks must be >= 1");
  L.n = b->n_seqs;
  L.maxb = b->max_blocks;
  L.T = 0;
  L.n_out = 0;
  for (int s = 0; s < L.n; ++s) {
    CHECK_ARG(b->q_len[s] >= 1, "batch: q_len must be >= 1");
    CHECK_ARG(b->ctx[s] >= 0, "batch: ctx must be >= 0");
    long end = (long)b->ctx[s] + b->q_len[s];
    CHECK_ARG(end <= (long)b->max_blocks * d->bt, "batch: block table too short for ctx + q_len");
    CHECK_ARG(end <= kMaxRope, "batch: position beyond RoPE table");
    for (int j = 0; j < (int)((end + d->bt - 1) / d->bt); ++j) {
      int blk = b->block_tables[(size_t)s * b->max_blocks + j];
      CHECK_ARG(blk >= 0 && blk < d->nblocks, "batch: block id out of range");
    }
    L.T += b->q_len[s];
    if (!b->want_token || b->want_token[s]) ++L.n_out;
  }
  CHECK_ARG(L.T <= d->max_T, "batch: sum(q_len) exceeds max_step_tokens");
  {
    // unique K/V bytes attended per layer + q in + o out
    const double kv_tok = 2.0 * d->cfg.n_kv_heads * d->cfg.head_dim * 2;
    double keys = 0;
    for (int s = 0; s < L.n; ++s) keys += (double)b->ctx[s] + b->q_len[s];
    L.attn_bytes = keys * kv_tok + 2.0 * L.T * d->cfg.n_q_heads * d->cfg.head_dim * 2;
  }
  for (int i = 0; i < L.T; ++i)
    CHECK_ARG(b->tokens[i] >= 0 && b->tokens[i] < d->cfg.vocab, "batch: token id out of range");
  const int G = d->cfg.n_q_heads / d->cfg.n_kv_heads;
  std::vector<int> seg_start;
  plan_attention(L.n, b->q_len, b->ctx, d->cfg.n_kv_heads, G, items, L.n_ws, L.n_dec, seg_start, L.n_pf);
  L.n_cta = seg_start.empty() ? 0 : (int)seg_start.size() - 1;
  L.n_items = (int)items.size();
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o = align_up(o + bytes, 16);
    return r;
  };
  L.off_qstart = take((L.n + 1) * 4);
  L.off_ctx = take(L.n * 4);
  L.off_tokens = take(L.T * 4);
  L.off_bt = take((size_t)L.n * L.maxb * 4);
  L.off_rowseq = take(L.T * 4);
  L.off_rowpos = take(L.T * 4);
  L.off_outrows = take(std::max(L.n_out, 1) * 4);
  L.off_items = take(items.size() * sizeof(AttnItem));
  L.off_seg = take(seg_start.size() * 4 + 4);
  L.total = o;
  int rc = ensure_meta(d, L.total);
  if (rc) return rc;
  rc = ensure_ws(d, L.n_ws);
  if (rc) return rc;
  uint8_t* h = d->h_meta;
  int32_t* qs = at<int32_t>(h, L.off_qstart);
  int32_t* rs = at<int32_t>(h, L.off_rowseq);
  int32_t* rp = at<int32_t>(h, L.off_rowpos);
  int32_t* orow = at<int32_t>(h, L.off_outrows);
  qs[0] = 0;
  int k = 0;
  for (int s = 0; s < L.n; ++s) {
    qs[s + 1] = qs[s] + b->q_len[s];
    for (int i = 0; i < b->q_len[s]; ++i) {
      rs[qs[s] + i] = s;
      rp[qs[s] + i] = b->ctx[s] + i;
    }
    if (!b->want_token || b->want_token[s]) orow[k++] = qs[s + 1] - 1;
  }
  std::memcpy(h + L.off_ctx, b->ctx, L.n * 4);
  std::memcpy(h + L.off_tokens, b->tokens, L.T * 4);
  std::memcpy(h + L.off_bt, b->block_tables, (size_t)L.n * L.maxb * 4);
  std::memcpy(h + L.off_items, items.data(), items.size() * sizeof(AttnItem));
  if (!seg_start.empty()) std::memcpy(h + L.off_seg, seg_start.data(), seg_start.size() * 4);
  return PPD_OK;
}

int run_attention(const ppd_model_cfg& c, const void* kv_map, const bf16* q, bf16* out,
                  const int* d_qstart, const int* d_ctx, const int* d_bt, int maxb,
                  const AttnItem* d_items, int n_dec, int n_items, const int* d_seg, int n_cta, int n_pf, int layer,
                  float* ws_o, float* ws_ml, int* counters, int* mix_ctr, cudaStream_t s) {
  AttnParams p{};
  p.seg_start = d_seg;
  p.items = d_items;
  p.q = q;
  p.out = out;
  p.q_start = d_qstart;
  p.ctx = d_ctx;
  p.block_tables = d_bt;
  p.max_blocks = maxb;
  p.n_layers = c.n_layers;
  p.layer = layer;
  p.n_q_heads = c.n_q_heads;
  p.n_kv_heads = c.n_kv_heads;
  p.group = c.n_q_heads / c.n_kv_heads;
  p.scale_log2 = (1.0f / std::sqrt((float)c.head_dim)) * 1.4426950408889634f;
  p.ws_o = ws_o;
  p.ws_ml = ws_ml;
  p.counters = counters;
  p.mix_ctr = mix_ctr;
  p.overlap = pdl_overlap();
  p.l2_hint = (gemm_tc_l2_hint() >> 1) & 1;
  // K2: a mixed step is ONE launch (prefill CTAs + decode CTAs)
  if (n_pf > 0) {
    CU(launch_mixed_attention(kv_map, p, d_items + n_dec, n_pf, (n_items - n_dec) * c.n_kv_heads, n_cta, s));
    return PPD_OK;
  }
  // decode rows: the balanced persistent kernel (n_cta > 0) or one CTA per item
  if (n_cta > 0) {
    CU(launch_decode_attention(kv_map, p, n_cta, p.group, s));
  } else if (n_dec > 0 && (attention_tc_enabled() || n_items == n_dec)) {
    CU(launch_paged_attention(kv_map, p, n_dec, s));
  }
  if (n_items > n_dec) {
    if (attention_tc_enabled()) {
      p.items = d_items + n_dec;
      if (g_attn_pf_persist)  // after the decode kernel on a mixed step that does not fit K2
        CU(launch_prefill_attention_persistent(kv_map, p, d_items + n_dec, n_items - n_dec, s));
      else
        CU(launch_prefill_attention_tc(kv_map, p, n_items - n_dec, s));
    } else if (n_cta > 0) {
      p.items = d_items + n_dec;
      CU(launch_paged_attention(kv_map, p, n_items - n_dec, s));
    } else {
      CU(launch_paged_attention(kv_map, p, n_items, s));  // decode + prefill items, one launch
    }
  }
  return PPD_OK;
}

bool layer_kernel_ok(const ppd_dev* d, int T);

void count_launches(ppd_dev* d, const StepLayout& L) {
  const long nl = d->cfg.n_layers;
  if (layer_kernel_ok(d, L.T)) {
    // embed, add_rmsnorm, qkv GEMM, rope_kv; per layer attention + K8; final norm, lm_head, argmax
    d->stats.own_launches += 2 * nl + 7;
  } else {
    // own kernels per layer: add_rmsnorm x2, rope_kv, attention, silu_mul; + embed, final norm, argmax
    d->stats.own_launches += 5 * nl + 3;
    d->stats.own_launches += 4 * nl + 1;  // tcgen05 GEMMs
  }
  d->stats.attn_launches += nl;
  d->stats.attn_bytes += L.attn_bytes * nl;
}

int prof_mark(ppd_dev* d, int kind, bool end) {
  if (!d->profiling) return PPD_OK;
  if (d->ev_used >= (int)d->ev_pool.size()) {
    cudaEvent_t e;
    CU(cudaEventCreate(&e));
    d->ev_pool.push_back(e);
  }
  if (!end) d->prof_marks.push_back({kind, d->ev_used});
  CU(cudaEventRecord(d->ev_pool[d->ev_used++], d->compute));
  return PPD_OK;
}

#define PROF(kind, end)                        \
  do {                                         \
    int _rc = prof_mark(d, kind, end);         \
    if (_rc) return _rc;                       \
  } while (0)

// Device-side usability of the K8 decode layer kernel for a step of T rows.
bool layer_kernel_ok(const ppd_dev* d, int T) {
  const ppd_model_cfg& c = d->cfg;
  if (!g_layer_kernel || T < 1 || T > 256 || T > 2 * device_sms()) return false;
  if (g_open_on_gpu[d->gpu].load() != 1) return false;
  if (c.d_model % 128 != 0 || c.d_model > 8192 || (2 * c.d_ff) % 128 != 0 || c.head_dim != 128) return false;
  const int W = (c.n_q_heads + 2 * c.n_kv_heads) * c.head_dim;
  const int max_sl = (int)std::min<size_t>(8, d->ws_rows / (size_t)T);
  LayerJob j;
  return layer_plan_job(j, d->proj32, T, c.d_model, c.n_q_heads * c.head_dim, device_sms(), max_sl) &&
         layer_plan_job(j, d->gu32, T, 2 * c.d_ff, c.d_model, device_sms(), max_sl) &&
         layer_plan_job(j, d->down32, T, c.d_model, c.d_ff, device_sms(), max_sl) &&
         layer_plan_job(j, d->qkv32, T, W, c.d_model, device_sms(), max_sl);
}

// Steps of <= 256 rows: per layer ONE attention launch + ONE K8 layer kernel
// (o -> add+norm -> gate|up -> SiLU -> down -> add+norm -> next qkv -> RoPE/KV).
// Same rounding points as the per-op path; the K-partial slices follow the
// grid-wide stream-K partition (deterministic slice order).
int forward_layers(ppd_dev* d, const StepLayout& L, int max_sl) {
  const ppd_model_cfg& c = d->cfg;
  cudaStream_t s = d->compute;
  const int Dh = c.head_dim, d_model = c.d_model, F = c.d_ff, T = L.T;
  const int qd = c.n_q_heads * Dh, kd = c.n_kv_heads * Dh, W = qd + 2 * kd;
  const int n_cta = device_sms();
  uint8_t* m = d->d_meta;
  const int* qstart = at<int>(m, L.off_qstart);
  const int* ctx = at<int>(m, L.off_ctx);
  const int* bt = at<int>(m, L.off_bt);
  const int* rowseq = at<int>(m, L.off_rowseq);
  const int* rowpos = at<int>(m, L.off_rowpos);
  const int* outrows = at<int>(m, L.off_outrows);
  const AttnItem* items = at<AttnItem>(m, L.off_items);
  int bn = 0, stages = 0, stage_bytes = 0, smem = 0;
  layer_shape(T, &bn, &stages, &stage_bytes, &smem);
  if (g_layer_stages > 0 && g_layer_stages < stages) {
    smem -= (stages - g_layer_stages) * stage_bytes;
    stages = g_layer_stages;
  }
  CU(cudaMemsetAsync(d->layer_sync, 0, (size_t)c.n_layers * 8 * sizeof(unsigned), s));
  // layer 0's qkv + RoPE/KV write through the per-op kernels
  GemmParts np_qkv, none;
  CU(launch_add_rmsnorm(d->x, nullptr, none, nullptr, d->ones, d->h, T, d_model, c.rms_eps, s));
  PROF(1, false);
  CU(gemm_run_split(d->h, d->layers[0].wqkv, d->qkv32, T, W, d_model, max_sl, &np_qkv, s));
  PROF(1, true);
  CU(launch_rope_kv_write(d->qkv32, np_qkv, d->layers[0].bqkv, rowseq, rowpos, bt, L.maxb, d->rope_cos,
                          d->rope_sin, d->q, d->kv, T, c.n_q_heads, c.n_kv_heads, Dh, c.n_layers, 0, d->bt, s));
  LayerParams p{};
  p.T = T;
  p.bn = bn;
  p.stages = stages;
  p.stage_bytes = stage_bytes;
  p.n_cta = n_cta;
  p.l2_ahead = g_layer_l2_ahead;

  p.x = d->x;
  p.h = d->h;
  p.m = d->m;
  p.norm_w = d->ones;
  p.eps = c.rms_eps;
  p.d_model = d_model;
  p.F = F;
  auto job = [&](int j, const bf16* wgt, const bf16* act, float* out, int N, int K) -> int {
    if (!layer_plan_job(p.job[j], out, T, N, K, n_cta, max_sl)) return fail(PPD_ERR_INVALID, "layer kernel plan");
    if (!gemm_tc_map(p.map_w[j], wgt, N, K, 128) || !gemm_tc_map(p.map_x[j], act, T, K, bn))
      return fail(PPD_ERR_CUDA, "cuTensorMapEncodeTiled failed (layer kernel)");
    return PPD_OK;
  };
  for (int l = 0; l < c.n_layers; ++l) {
    const Layer& w = d->layers[l];
    PROF(0, false);
    int rc = run_attention(c, d->kv_map, d->q, d->attn, qstart, ctx, bt, L.maxb, items, L.n_dec, L.n_items,
                           at<int>(m, L.off_seg), L.n_cta, L.n_pf, l, d->ws_o, d->ws_ml, d->counters,
                           d->counters + (size_t)d->max_S * c.n_kv_heads, s);
    if (rc) return rc;
    PROF(0, true);
    const bool next = l + 1 < c.n_layers;
    p.n_jobs = next ? 4 : 3;
    p.sync = d->layer_sync + (size_t)l * 8;
    if ((rc = job(0, w.wo, d->attn, d->proj32, d_model, qd)) || (rc = job(1, w.wgu, d->h, d->gu32, 2 * F, d_model)) ||
        (rc = job(2, w.wdown, d->m, d->down32, d_model, F)))
      return rc;
    if (next) {
      const Layer& wn = d->layers[l + 1];
      if ((rc = job(3, wn.wqkv, d->h, d->qkv32, W, d_model))) return rc;
      p.rope = RopeArgs{d->qkv32, p.job[3].parts, wn.bqkv, rowseq, rowpos, bt, L.maxb, d->rope_cos, d->rope_sin,
                        d->q, d->kv, c.n_q_heads, c.n_kv_heads, Dh, c.n_layers, l + 1, d->bt};
    }
    PROF(1, false);
    CU(launch_decode_layer(p, smem, s));
    PROF(1, true);
  }
  count_launches(d, L);
  GemmParts none2;
  CU(launch_final_norm(d->x, nullptr, none2, nullptr, outrows, L.n_out, d->ones, d->hl, T, d_model, c.rms_eps, s));
  CU(gemm_run(d->hl, d->lm_head, d->logits, L.n_out, c.vocab, d_model, true, s));
  CU(launch_argmax(d->logits, L.n_out, c.vocab, d->d_tokens_out, s));
  return PPD_OK;
}

// The forward pass of one step; metadata already staged in d->d_meta.
int forward(ppd_dev* d, const StepLayout& L) {
  const ppd_model_cfg& c = d->cfg;
  cudaStream_t s = d->compute;
  const int Dh = c.head_dim, d_model = c.d_model, F = c.d_ff;
  const int qd = c.n_q_heads * Dh, kd = c.n_kv_heads * Dh, W = qd + 2 * kd;
  uint8_t* m = d->d_meta;
  const int* qstart = at<int>(m, L.off_qstart);
  const int* ctx = at<int>(m, L.off_ctx);
  const int* tokens = at<int>(m, L.off_tokens);
  const int* bt = at<int>(m, L.off_bt);
  const int* rowseq = at<int>(m, L.off_rowseq);
  const int* rowpos = at<int>(m, L.off_rowpos);
  const int* outrows = at<int>(m, L.off_outrows);
  const AttnItem* items = at<AttnItem>(m, L.off_items);
  const int T = L.T;
  // K-partial slices the fp32 workspaces hold for this step (Tp token rows of slices)
  const int max_sl = std::max(1, std::min(8, (int)(d->ws_rows / (size_t)std::max(T, 1))));
  GemmParts np_down;

  CU(launch_embed(tokens, d->embed, d->x, T, d_model, s));
  if (layer_kernel_ok(d, T)) return forward_layers(d, L, max_sl);
  for (int l = 0; l < c.n_layers; ++l) {
    GemmParts np_qkv, np_o;
    const Layer& w = d->layers[l];
    // x += down(prev) ; h = norm(x)
    CU(launch_add_rmsnorm(d->x, l == 0 ? nullptr : d->down32, np_down, nullptr, d->ones, d->h, T, d_model,
                          c.rms_eps, s));
    PROF(1, false);
    CU(gemm_run_split(d->h, w.wqkv, d->qkv32, T, W, d_model, max_sl, &np_qkv, s));
    PROF(1, true);
    CU(launch_rope_kv_write(d->qkv32, np_qkv, w.bqkv, rowseq, rowpos, bt, L.maxb, d->rope_cos,
                            d->rope_sin, d->q, d->kv, T, c.n_q_heads, c.n_kv_heads, Dh, c.n_layers,
                            l, d->bt, s));
    PROF(0, false);
    int rc = run_attention(c, d->kv_map, d->q, d->attn, qstart, ctx, bt, L.maxb, items, L.n_dec, L.n_items,
                           at<int>(m, L.off_seg), L.n_cta, L.n_pf, l, d->ws_o, d->ws_ml, d->counters,
                           d->counters + (size_t)d->max_S * c.n_kv_heads, s);
    if (rc) return rc;
    PROF(0, true);
    PROF(1, false);
    CU(gemm_run_split(d->attn, w.wo, d->proj32, T, d_model, qd, max_sl, &np_o, s));
    PROF(1, true);
    CU(launch_add_rmsnorm(d->x, d->proj32, np_o, nullptr, d->ones, d->h, T, d_model, c.rms_eps, s));
    PROF(1, false);
    if (g_mlp_fused == 1 || (g_mlp_fused == 2 && T >= kMlpFusedMinRows)) {
      CU(gemm_run_silu(d->h, w.wgu, d->m, T, 2 * F, d_model, s));
      PROF(1, true);
    } else {
      GemmParts np_gu;
      CU(gemm_run_split(d->h, w.wgu, d->gu32, T, 2 * F, d_model, max_sl, &np_gu, s));
      PROF(1, true);
      CU(launch_silu_mul(d->gu32, np_gu, d->m, T, F, s));
    }
    PROF(1, false);
    CU(gemm_run_split(d->m, w.wdown, d->down32, T, d_model, F, max_sl, &np_down, s));
    PROF(1, true);
  }
  count_launches(d, L);
  CU(launch_final_norm(d->x, d->down32, np_down, nullptr, outrows, L.n_out, d->ones, d->hl, T, d_model,
                       c.rms_eps, s));
  CU(gemm_run(d->hl, d->lm_head, d->logits, L.n_out, c.vocab, d_model, true, s));
  CU(launch_argmax(d->logits, L.n_out, c.vocab, d->d_tokens_out, s));
  return PPD_OK;
}

int alloc_workspaces(ppd_dev* d) {
  const ppd_model_cfg& c = d->cfg;
  const size_t T = d->max_T, S = d->max_S;
  const size_t qd = (size_t)c.n_q_heads * c.head_dim, kd = (size_t)c.n_kv_heads * c.head_dim;
  CU(cudaMalloc(&d->x, T * c.d_model * 2));
  CU(cudaMalloc(&d->h, T * c.d_model * 2));
  CU(cudaMalloc(&d->q, T * qd * 2));
  CU(cudaMalloc(&d->attn, T * qd * 2));
  CU(cudaMalloc(&d->m, T * c.d_ff * 2));
  CU(cudaMalloc(&d->hl, S * c.d_model * 2));
  // fp32 GEMM outputs also hold up to 8 K-split partial slices of a <=256-token
  // step and 2 of a full-size step: prefill-size o / down GEMMs (N = 4096 -> 32
  // weight tiles x T/256 token tiles) need a balanced 2-way K split to fill
  // the 148 SMs (1.3 waves of tiles otherwise at T = 1536)
  const size_t Tp = std::max<size_t>(g_ws_two_slices ? 2 * T : T, 8 * 256);
  d->ws_rows = Tp;
  CU(cudaMalloc(&d->qkv32, Tp * (qd + 2 * kd) * 4));
  CU(cudaMalloc(&d->proj32, Tp * c.d_model * 4));
  CU(cudaMalloc(&d->gu32, Tp * 2 * c.d_ff * 4));
  CU(cudaMalloc(&d->down32, Tp * c.d_model * 4));
  CU(cudaMalloc(&d->logits, S * c.vocab * 4));
  CU(cudaMalloc(&d->layer_sync, (size_t)c.n_layers * 8 * sizeof(unsigned)));
  // split-merge counters [S][Hkv] + the K2 queue heads / done counter [4]
  CU(cudaMalloc(&d->counters, (S * c.n_kv_heads + 4) * 4));
  CU(cudaMemset(d->counters, 0, (S * c.n_kv_heads + 4) * 4));
  CU(cudaMallocHost(&d->h_tokens_out, S * 4));
  CU(cudaMalloc(&d->d_tokens_out, S * 4));
  // RoPE cos/sin table, built in double on the host (same recipe as the oracle)
  const int half = c.head_dim / 2;
  std::vector<float> cs((size_t)kMaxRope * half), sn((size_t)kMaxRope * half);
  std::vector<double> inv(half);
  for (int i = 0; i < half; ++i) inv[i] = std::pow((double)c.rope_theta, -2.0 * i / (double)c.head_dim);
  for (int p = 0; p < kMaxRope; ++p)
    for (int i = 0; i < half; ++i) {
      double a = (double)p * inv[i];
      cs[(size_t)p * half + i] = (float)std::cos(a);
      sn[(size_t)p * half + i] = (float)std::sin(a);
    }
  CU(cudaMalloc(&d->rope_cos, cs.size() * 4));
  CU(cudaMalloc(&d->rope_sin, sn.size() * 4));
  CU(cudaMemcpy(d->rope_cos, cs.data(), cs.size() * 4, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(d->rope_sin, sn.data(), sn.size() * 4, cudaMemcpyHostToDevice));
  return PPD_OK;
}

std::mutex g_weights_mu;
std::vector<SharedWeights*> g_weights;

bool same_cfg(const ppd_model_cfg& a, const ppd_model_cfg& b) { return std::memcmp(&a, &b, sizeof(a)) == 0; }

void release_weights(ppd_dev* d) {
  if (!d->wshared) return;
  std::lock_guard<std::mutex> lk(g_weights_mu);
  SharedWeights* w = d->wshared;
  d->wshared = nullptr;
  if (--w->refs > 0) return;
  cudaFree(w->mem);
  g_weights.erase(std::find(g_weights.begin(), g_weights.end(), w));
  delete w;
}

void free_all(ppd_dev* d) {
  release_weights(d);
  for (CopySlot& c : d->copy) {
    if (c.e0) cudaEventDestroy(c.e0);
    if (c.e1) cudaEventDestroy(c.e1);
    if (c.h_bt) cudaFreeHost(c.h_bt);
    if (c.d_bt) cudaFree(c.d_bt);
    c = CopySlot{};
  }
  void* dev_ptrs[] = {d->kv, d->x, d->h, d->q, d->attn, d->m, d->hl, d->qkv32, d->proj32,
                      d->gu32, d->down32, d->logits, d->layer_sync, d->ws_o, d->ws_ml, d->counters, d->d_meta,
                      d->d_tokens_out, d->rope_cos, d->rope_sin};
  for (void* p : dev_ptrs)
    if (p) cudaFree(p);
  if (d->h_meta) cudaFreeHost(d->h_meta);
  if (d->h_tokens_out) cudaFreeHost(d->h_tokens_out);
  cudaEvent_t evs[] = {d->ev0, d->ev1, d->compute_done};
  for (auto e : evs)
    if (e) cudaEventDestroy(e);
  for (auto e : d->ev_pool) cudaEventDestroy(e);
  clear_graphs(d);
  if (d->compute) cudaStreamDestroy(d->compute);
  if (d->xfer) cudaStreamDestroy(d->xfer);
}

}  // namespace

// ============================================================ C-ABI
extern "C" {

const char* ppd_last_error(void) { return g_err.c_str(); }
int ppd_version(void) { return 1; }

int ppd_device_count(int32_t* n) {
  int c = 0;
  CU(cudaGetDeviceCount(&c));
  *n = c;
  return PPD_OK;
}

int ppd_kv_block_bytes(const ppd_model_cfg* cfg, int32_t block_tokens, uint64_t* bytes) {
  int rc = validate_cfg(cfg);
  if (rc) return rc;
  CHECK_ARG(block_tokens == 16, "block_tokens must be 16");
  *bytes = (uint64_t)cfg->n_layers * 2 * cfg->n_kv_heads * block_tokens * cfg->head_dim * 2;
  return PPD_OK;
}

int ppd_dev_open(int32_t gpu, const ppd_model_cfg* cfg, int32_t max_step_tokens,
                 int32_t max_step_seqs, ppd_dev** out) {
  int rc = validate_cfg(cfg);
  if (rc) return rc;
  CHECK_ARG(out, "null out");
  CHECK_ARG(max_step_tokens >= 1 && max_step_seqs >= 1 && max_step_seqs <= max_step_tokens,
            "max_step_tokens/max_step_seqs invalid");
  int ndev = 0;
  CU(cudaGetDeviceCount(&ndev));
  CHECK_ARG(gpu >= 0 && gpu < ndev, "gpu index out of range");
  CU(cudaSetDevice(gpu));
  ppd_dev* d = new ppd_dev();
  d->gpu = gpu;
  d->cfg = *cfg;
  d->max_T = max_step_tokens;
  d->max_S = max_step_seqs;
  if (const char* g = std::getenv("PPD_GRAPHS")) d->use_graphs = std::strcmp(g, "0") != 0;
  auto bail = [&](int code) {
    free_all(d);
    delete d;
    return code;
  };
  if (cudaStreamCreateWithFlags(&d->compute, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&d->xfer, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&d->ev0) != cudaSuccess || cudaEventCreate(&d->ev1) != cudaSuccess ||
      cudaEventCreateWithFlags(&d->compute_done, cudaEventDisableTiming) != cudaSuccess)
    return bail(fail(PPD_ERR_CUDA, "stream/event creation failed"));
  rc = alloc_workspaces(d);
  if (rc) return bail(rc);
  g_open_on_gpu[gpu].fetch_add(1);
  *out = d;
  return PPD_OK;
}

int ppd_dev_close(ppd_dev* d) {
  if (!d) return PPD_OK;
  cudaSetDevice(d->gpu);
  cudaDeviceSynchronize();
  g_open_on_gpu[d->gpu].fetch_sub(1);
  free_all(d);
  delete d;
  return PPD_OK;
}

int ppd_load_random_weights(ppd_dev* d, uint64_t seed) {
  CHECK_ARG(d, "null dev");
  CU(cudaSetDevice(d->gpu));
  const ppd_model_cfg& c = d->cfg;
  const size_t dm = c.d_model, F = c.d_ff, V = c.vocab;
  const size_t qd = (size_t)c.n_q_heads * c.head_dim, kd = (size_t)c.n_kv_heads * c.head_dim;
  const size_t per_layer = align_up((qd + 2 * kd) * dm * 2, 256) + align_up(dm * qd * 2, 256) +
                           align_up(2 * F * dm * 2, 256) + align_up(dm * F * 2, 256) +
                           align_up((qd + 2 * kd) * 4, 256);
  const size_t total = 2 * align_up(V * dm * 2, 256) + align_up(dm * 2, 256) + per_layer * c.n_layers;
  std::lock_guard<std::mutex> lk(g_weights_mu);
  SharedWeights* w = nullptr;
  for (SharedWeights* e : g_weights)
    if (e->gpu == d->gpu && e->seed == seed && same_cfg(e->cfg, c)) w = e;
  const bool fresh = w == nullptr;
  if (d->wshared && d->wshared != w) {  // re-seeding: drop the old set first
    SharedWeights* old = d->wshared;
    d->wshared = nullptr;
    if (--old->refs == 0) {
      cudaFree(old->mem);
      g_weights.erase(std::find(g_weights.begin(), g_weights.end(), old));
      delete old;
    }
  }
  if (fresh) {
    w = new SharedWeights{d->gpu, c, seed, nullptr, total, 0};
    if (cudaMalloc(&w->mem, total) != cudaSuccess) {
      cudaGetLastError();
      delete w;
      return fail(PPD_ERR_OOM, "weights: cudaMalloc of " + std::to_string(total) + " bytes failed");
    }
    g_weights.push_back(w);
  }
  if (d->wshared != w) {
    d->wshared = w;
    w->refs += 1;
  }
  uint8_t* p = static_cast<uint8_t*>(w->mem);
  auto take = [&](size_t bytes) {
    uint8_t* r = p;
    p += align_up(bytes, 256);
    return r;
  };
  cudaStream_t s = d->compute;
  d->embed = reinterpret_cast<bf16*>(take(V * dm * 2));
  d->lm_head = reinterpret_cast<bf16*>(take(V * dm * 2));
  d->ones = reinterpret_cast<bf16*>(take(dm * 2));
  if (fresh) {
    CU(launch_fill_random(d->embed, V * dm, seed, 0, 0, s));
    CU(launch_fill_matrix(d->lm_head, V, dm, seed, 8, 0, s));
    CU(launch_fill_const(d->ones, dm, 1.0f, s));
  }
  d->layers.assign(c.n_layers, Layer{});
  for (int l = 0; l < c.n_layers; ++l) {
    Layer& lw = d->layers[l];
    lw.wqkv = reinterpret_cast<bf16*>(take((qd + 2 * kd) * dm * 2));
    lw.wo = reinterpret_cast<bf16*>(take(dm * qd * 2));
    lw.wgu = reinterpret_cast<bf16*>(take(2 * F * dm * 2));
    lw.wdown = reinterpret_cast<bf16*>(take(dm * F * 2));
    float* b = reinterpret_cast<float*>(take((qd + 2 * kd) * 4));
    lw.bqkv = c.qkv_bias ? b : nullptr;
    if (!fresh) continue;
    CU(launch_fill_qkv(lw.wqkv, (int)qd, (int)kd, (int)dm, seed, l, s));
    CU(launch_fill_matrix(lw.wo, dm, qd, seed, 4, l, s));
    CU(launch_fill_gate_up(lw.wgu, (int)F, (int)dm, seed, l, s));
    CU(launch_fill_matrix(lw.wdown, dm, F, seed, 7, l, s));
    if (c.qkv_bias) CU(launch_fill_bias(lw.bqkv, (int)qd, (int)kd, seed, l, s));
  }
  CU(cudaStreamSynchronize(s));
  d->weights_ready = true;
  return PPD_OK;
}

int ppd_weights_info(ppd_dev* d, uint64_t* bytes, int32_t* shared_by) {
  CHECK_ARG(d && bytes && shared_by, "null arg");
  std::lock_guard<std::mutex> lk(g_weights_mu);
  *bytes = d->wshared ? d->wshared->bytes : 0;
  *shared_by = d->wshared ? d->wshared->refs : 0;
  return PPD_OK;
}

int ppd_kv_pool_init(ppd_dev* d, int32_t block_tokens, int32_t num_blocks) {
  CHECK_ARG(d, "null dev");
  CHECK_ARG(block_tokens == 16, "block_tokens must be 16");
  CHECK_ARG(num_blocks >= 1, "num_blocks must be >= 1");
  CU(cudaSetDevice(d->gpu));
  uint64_t bb = 0;
  int rc = ppd_kv_block_bytes(&d->cfg, block_tokens, &bb);
  if (rc) return rc;
  uint64_t rows = (uint64_t)num_blocks * d->cfg.n_layers * 2 * d->cfg.n_kv_heads * block_tokens;
  CHECK_ARG(rows < (1ull << 31), "KV pool too large for 32-bit TMA row coordinates");
  if (d->kv) cudaFree(d->kv);
  d->kv = nullptr;
  CU(cudaMalloc(&d->kv, bb * num_blocks));
  CU(cudaMemset(d->kv, 0, bb * num_blocks));
  d->bt = block_tokens;
  d->nblocks = num_blocks;
  d->kv_bytes = bb * num_blocks;
  if (make_kv_tensor_map(d->kv_map, d->kv, rows) != 0)
    return fail(PPD_ERR_CUDA, "cuTensorMapEncodeTiled failed for the KV pool");
  return PPD_OK;
}

int ppd_kv_pool_ptr(ppd_dev* d, void** ptr, uint64_t* bytes) {
  CHECK_ARG(d && ptr && bytes, "null arg");
  *ptr = d->kv;
  *bytes = d->kv_bytes;
  return PPD_OK;
}

int ppd_kv_pool_write(ppd_dev* d, uint64_t offset, const void* host, uint64_t bytes) {
  CHECK_ARG(d && host, "null arg");
  CHECK_ARG(d->kv, "KV pool not initialised");
  CHECK_ARG(offset <= d->kv_bytes && bytes <= d->kv_bytes - offset, "range outside the KV pool");
  CU(cudaSetDevice(d->gpu));
  CU(cudaStreamSynchronize(d->compute));
  CU(cudaMemcpy(reinterpret_cast<uint8_t*>(d->kv) + offset, host, bytes, cudaMemcpyHostToDevice));
  return PPD_OK;
}

int ppd_kv_pool_read(ppd_dev* d, uint64_t offset, void* host, uint64_t bytes) {
  CHECK_ARG(d && host, "null arg");
  CHECK_ARG(d->kv, "KV pool not initialised");
  CHECK_ARG(offset <= d->kv_bytes && bytes <= d->kv_bytes - offset, "range outside the KV pool");
  CU(cudaSetDevice(d->gpu));
  CU(cudaStreamSynchronize(d->compute));
  CU(cudaStreamSynchronize(d->xfer));
  CU(cudaMemcpy(host, reinterpret_cast<const uint8_t*>(d->kv) + offset, bytes, cudaMemcpyDeviceToHost));
  return PPD_OK;
}

int ppd_step_submit(ppd_dev* d, const ppd_batch* b) {
  CHECK_ARG(d, "null dev");
  if (!d->weights_ready || !d->kv) return fail(PPD_ERR_STATE, "step before weights and KV pool");
  if (d->pending) return fail(PPD_ERR_STATE, "step already in flight");
  CU(cudaSetDevice(d->gpu));
  StepLayout L{};
  std::vector<AttnItem> items;
  int rc = pack_batch(d, b, L, items);
  if (rc) return rc;
  CU(cudaMemcpyAsync(d->d_meta, d->h_meta, L.total, cudaMemcpyHostToDevice, d->compute));
  CU(cudaEventRecord(d->ev0, d->compute));
  // repeated shapes replay a captured graph (decode steps: ~300 launches -> 1)
  // every launch parameter of forward() is a function of these (grids: items, n_dec, n_cta)
  const ppd_dev::GraphKey key{L.n, L.T, L.maxb, L.n_out, L.n_items * 4096 + L.n_dec,
                             ((long long)L.n_ws * 8192 + L.n_cta) * 256 + L.n_pf, layer_kernel_ok(d, L.T) ? 1 : 0};
  if (d->tuning_epoch != g_tuning_epoch) {  // kernels chosen at capture time changed
    clear_graphs(d);
    d->tuning_epoch = g_tuning_epoch;
  }
  const bool graph_ok = d->use_graphs && !d->profiling && d->shape_seen[key]++ > 0;
  if (graph_ok) {
    auto it = d->graphs.find(key);
    if (it == d->graphs.end()) {
      if (d->graphs.size() >= 64) clear_graphs(d);
      cudaGraph_t g = nullptr;
      CU(cudaStreamBeginCapture(d->compute, cudaStreamCaptureModeThreadLocal));
      const ppd_dev_stats saved = d->stats;
      rc = forward(d, L);
      d->stats = saved;  // launches are counted when the graph runs
      cudaError_t ce = cudaStreamEndCapture(d->compute, &g);
      if (rc) return rc;
      CU(ce);
      cudaGraphExec_t ge = nullptr;
      CU(cudaGraphInstantiate(&ge, g, 0));
      cudaGraphDestroy(g);
      it = d->graphs.emplace(key, ge).first;
    }
    CU(cudaGraphLaunch(it->second, d->compute));
    count_launches(d, L);
  } else {
    rc = forward(d, L);
    if (rc) return rc;
  }
  CU(cudaEventRecord(d->ev1, d->compute));
  CU(cudaMemcpyAsync(d->h_tokens_out, d->d_tokens_out, L.n_out * 4, cudaMemcpyDeviceToHost,
                     d->compute));
  CU(cudaEventRecord(d->compute_done, d->compute));
  d->pending = L.n_out > 0 ? L.n_out : -1;
  d->last_logit_rows = L.n_out;
  return PPD_OK;
}

int ppd_step_wait(ppd_dev* d, int32_t* out_tokens, float* out_ms) {
  CHECK_ARG(d, "null dev");
  if (!d->pending) return fail(PPD_ERR_STATE, "no step in flight");
  CU(cudaSetDevice(d->gpu));
  CU(cudaEventSynchronize(d->compute_done));
  int n = d->pending > 0 ? d->pending : 0;
  d->pending = 0;
  if (out_tokens && n) std::memcpy(out_tokens, d->h_tokens_out, n * 4);
  float ms = 0.f;
  CU(cudaEventElapsedTime(&ms, d->ev0, d->ev1));
  if (out_ms) *out_ms = ms;
  d->stats.steps += 1;
  d->stats.step_ms += ms;
  for (auto& mk : d->prof_marks) {
    float t = 0.f;
    CU(cudaEventElapsedTime(&t, d->ev_pool[mk.second], d->ev_pool[mk.second + 1]));
    (mk.first == 0 ? d->stats.attn_ms : d->stats.gemm_ms) += t;
  }
  d->prof_marks.clear();
  d->ev_used = 0;
  return PPD_OK;
}

int ppd_dev_set_profiling(ppd_dev* d, int32_t on) {
  CHECK_ARG(d, "null dev");
  if (d->pending) return fail(PPD_ERR_STATE, "cannot toggle profiling with a step in flight");
  d->profiling = on != 0;
  return PPD_OK;
}

int ppd_dev_get_stats(ppd_dev* d, ppd_dev_stats* out) {
  CHECK_ARG(d && out, "null arg");
  *out = d->stats;
  return PPD_OK;
}

int ppd_dev_reset_stats(ppd_dev* d) {
  CHECK_ARG(d, "null dev");
  d->stats = ppd_dev_stats{};
  return PPD_OK;
}

int ppd_step(ppd_dev* d, const ppd_batch* b, int32_t* out_tokens, float* out_ms) {
  int rc = ppd_step_submit(d, b);
  if (rc) return rc;
  return ppd_step_wait(d, out_tokens, out_ms);
}

int ppd_last_logits(ppd_dev* d, float* out, int64_t max_floats) {
  CHECK_ARG(d && out, "null arg");
  int64_t n = (int64_t)d->last_logit_rows * d->cfg.vocab;
  CHECK_ARG(n <= max_floats, "output buffer too small");
  CU(cudaSetDevice(d->gpu));
  CU(cudaMemcpy(out, d->logits, n * 4, cudaMemcpyDeviceToHost));
  return PPD_OK;
}

int ppd_prefill(ppd_dev* d, int32_t kind, const int32_t* tokens, int32_t n_new, int32_t n_ctx,
                const int32_t* block_table, int32_t n_blocks, int32_t* out_token, float* out_ms) {
  // mirrors the reference's argument checks (costmodel.cpp:319, :325-327)
  if (kind == PPD_PREFILL_FULL) {
    CHECK_ARG(n_new >= 1, "full_prefill_time: n must be >= 1");
    CHECK_ARG(n_ctx == 0, "full prefill recomputes the whole history: n_ctx must be 0");
  } else if (kind == PPD_PREFILL_APPEND) {
    CHECK_ARG(n_new >= 1, "append_prefill_time: m must be >= 1");
    CHECK_ARG(n_ctx >= 0, "append_prefill_time: n_ctx must be >= 0");
  } else {
    return fail(PPD_ERR_INVALID, "unknown prefill kind");
  }
  ppd_batch b{};
  b.n_seqs = 1;
  b.q_len = &n_new;
  b.ctx = &n_ctx;
  b.tokens = tokens;
  b.block_tables = block_table;
  b.max_blocks = n_blocks;
  b.want_token = nullptr;
  return ppd_step(d, &b, out_token, out_ms);
}

int ppd_kv_copy_submit(ppd_dev* src, ppd_dev* dst, const int32_t* src_block_table,
                       const int32_t* dst_block_table, int32_t n_blocks, int32_t start, int32_t n_tokens,
                       uint64_t* ticket) {
  // reference: kv_transfer_time requires tokens >= 1 (costmodel.cpp:335)
  CHECK_ARG(src && dst && ticket, "null arg");
  CHECK_ARG(n_tokens >= 1, "kv_transfer_time: tokens >= 1");
  CHECK_ARG(n_blocks >= 1 && src_block_table && dst_block_table, "empty block tables");
  CHECK_ARG(start >= 0 && (long)start + n_tokens <= (long)n_blocks * dst->bt, "token range outside block table");
  CHECK_ARG(src->kv && dst->kv && src->bt == dst->bt, "pools not initialised / block size mismatch");
  CHECK_ARG(same_cfg(src->cfg, dst->cfg), "source and destination model shapes differ");
  for (int j = start / dst->bt; j <= (start + n_tokens - 1) / dst->bt; ++j) {
    CHECK_ARG(src_block_table[j] >= 0 && src_block_table[j] < src->nblocks, "src block id out of range");
    CHECK_ARG(dst_block_table[j] >= 0 && dst_block_table[j] < dst->nblocks, "dst block id out of range");
  }
  const uint64_t t = dst->copy_head.load(std::memory_order_relaxed);
  if (t - dst->copy_done.load(std::memory_order_acquire) >= (uint64_t)kCopySlots)
    return fail(PPD_ERR_STATE, "too many KV copies in flight into this device (wait for older tickets)");
  CU(cudaSetDevice(dst->gpu));
  if (src->gpu != dst->gpu && !(dst->peer_mask & (1ull << src->gpu))) {
    // the copy kernel runs on the destination and pulls from the source pool over NVLink
    cudaError_t e = cudaDeviceEnablePeerAccess(src->gpu, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
      return fail(PPD_ERR_CUDA, std::string("peer access: ") + cudaGetErrorString(e));
    cudaGetLastError();
    dst->peer_mask |= 1ull << src->gpu;
  }
  CopySlot& c = dst->copy[t % kCopySlots];
  if (!c.e0) {
    CU(cudaEventCreate(&c.e0));
    CU(cudaEventCreate(&c.e1));
  }
  if (c.cap < n_blocks) {  // grows rarely (first hops / longer contexts); never per copy
    if (c.h_bt) cudaFreeHost(c.h_bt);
    if (c.d_bt) cudaFree(c.d_bt);
    c.h_bt = nullptr;
    c.d_bt = nullptr;
    c.cap = 0;
    const int cap = std::max(n_blocks, 1024);
    CU(cudaMallocHost(&c.h_bt, (size_t)cap * 2 * 4));
    CU(cudaMalloc(&c.d_bt, (size_t)cap * 2 * 4));
    c.cap = cap;
  }
  std::memcpy(c.h_bt, src_block_table, (size_t)n_blocks * 4);
  std::memcpy(c.h_bt + n_blocks, dst_block_table, (size_t)n_blocks * 4);
  // the producer's KV must be complete: fence after the source's last submitted step
  CU(cudaStreamWaitEvent(dst->xfer, src->compute_done, 0));
  CU(cudaEventRecord(c.e0, dst->xfer));
  CU(cudaMemcpyAsync(c.d_bt, c.h_bt, (size_t)n_blocks * 2 * 4, cudaMemcpyHostToDevice, dst->xfer));
  KvCopyParams p{};
  p.src_pool = src->kv;
  p.dst_pool = dst->kv;
  p.src_blocks = c.d_bt;
  p.dst_blocks = c.d_bt + n_blocks;
  p.start = start;
  p.n_tokens = n_tokens;
  p.n_layers = dst->cfg.n_layers;
  p.n_kv_heads = dst->cfg.n_kv_heads;
  p.block_tokens = dst->bt;
  p.head_dim = dst->cfg.head_dim;
  CU(launch_kv_copy(p, dst->xfer));
  CU(cudaEventRecord(c.e1, dst->xfer));
  dst->copy_head.store(t + 1, std::memory_order_release);
  *ticket = t;
  return PPD_OK;
}

int ppd_kv_copy_wait(ppd_dev* dst, uint64_t ticket, float* out_ms) {
  CHECK_ARG(dst, "null dev");
  const uint64_t done = dst->copy_done.load(std::memory_order_acquire);
  CHECK_ARG(ticket == done && ticket < dst->copy_head.load(std::memory_order_acquire),
            "tickets must be waited for once each, in submission order");
  CU(cudaSetDevice(dst->gpu));
  CopySlot& c = dst->copy[ticket % kCopySlots];
  CU(cudaEventSynchronize(c.e1));
  if (out_ms) CU(cudaEventElapsedTime(out_ms, c.e0, c.e1));
  dst->copy_done.store(ticket + 1, std::memory_order_release);
  return PPD_OK;
}

int ppd_kv_copy(ppd_dev* src, ppd_dev* dst, const int32_t* src_block_table,
                const int32_t* dst_block_table, int32_t n_blocks, int32_t start, int32_t n_tokens,
                float* out_ms) {
  CHECK_ARG(dst, "null dev");
  // earlier asynchronous hops into dst complete first (tickets retire in order)
  while (dst->copy_done.load() < dst->copy_head.load()) {
    int rc = ppd_kv_copy_wait(dst, dst->copy_done.load(), nullptr);
    if (rc) return rc;
  }
  uint64_t t = 0;
  int rc = ppd_kv_copy_submit(src, dst, src_block_table, dst_block_table, n_blocks, start, n_tokens, &t);
  if (rc) return rc;
  return ppd_kv_copy_wait(dst, t, out_ms);
}

// Peer bandwidth probe (bench.py, N > 1): bytes copied from src_gpu to
// dst_gpu per second, best of `iters`. mode 0: copy engines
// (cudaMemcpyPeerAsync); mode 1: an SM pull kernel on dst reading src over
// NVLink (the K7 access pattern: 16 B loads, streaming stores).
int ppd_p2p_bandwidth(int32_t src_gpu, int32_t dst_gpu, uint64_t bytes, int32_t iters, int32_t mode,
                      double* gbs) {
  CHECK_ARG(gbs && iters >= 1 && bytes >= 16 && bytes % 16 == 0 && (mode == 0 || mode == 1), "bad args");
  int ndev = 0;
  CU(cudaGetDeviceCount(&ndev));
  CHECK_ARG(src_gpu >= 0 && src_gpu < ndev && dst_gpu >= 0 && dst_gpu < ndev, "gpu index out of range");
  void *a = nullptr, *b = nullptr;
  CU(cudaSetDevice(src_gpu));
  CU(cudaMalloc(&a, bytes));
  CU(cudaMemset(a, 1, bytes));
  CU(cudaDeviceSynchronize());
  CU(cudaSetDevice(dst_gpu));
  if (src_gpu != dst_gpu) {
    cudaError_t e = cudaDeviceEnablePeerAccess(src_gpu, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
      cudaFree(a);
      return fail(PPD_ERR_CUDA, std::string("peer access: ") + cudaGetErrorString(e));
    }
    cudaGetLastError();
  }
  cudaStream_t st = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  int rc = PPD_OK;
  double best = 0;
  if (cudaMalloc(&b, bytes) != cudaSuccess || cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) {
    rc = fail(PPD_ERR_CUDA, "p2p probe: allocation failed");
  } else {
    for (int i = 0; i <= iters && rc == PPD_OK; ++i) {  // iteration 0 warms up
      cudaEventRecord(e0, st);
      cudaError_t e = mode == 0 ? cudaMemcpyPeerAsync(b, dst_gpu, a, src_gpu, bytes, st)
                                : launch_pull_copy(static_cast<const uint4*>(a), static_cast<uint4*>(b), bytes / 16, st);
      cudaEventRecord(e1, st);
      if (e == cudaSuccess) e = cudaEventSynchronize(e1);
      if (e != cudaSuccess) {
        rc = fail(PPD_ERR_CUDA, std::string("p2p probe: ") + cudaGetErrorString(e));
        break;
      }
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (i > 0 && ms > 0) best = std::max(best, (double)bytes / (ms * 1e-3) / 1e9);
    }
  }
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (st) cudaStreamDestroy(st);
  if (b) cudaFree(b);
  cudaSetDevice(src_gpu);
  cudaFree(a);
  *gbs = best;
  return rc;
}

// ------------------------------------------------------------ test entry points
int ppd_op_attention(const ppd_model_cfg* cfg, const void* q, const void* kv_pool,
                     int32_t num_blocks, int32_t block_tokens, int32_t layer, int32_t n_seqs,
                     const int32_t* q_start, const int32_t* ctx, const int32_t* block_tables,
                     int32_t max_blocks, void* out, void* stream) {
  int rc = validate_cfg(cfg);
  if (rc) return rc;
  CHECK_ARG(block_tokens == 16, "block_tokens must be 16");
  CHECK_ARG(n_seqs >= 1 && layer >= 0 && layer < cfg->n_layers, "bad n_seqs/layer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<int32_t> qlen(n_seqs);
  for (int i = 0; i < n_seqs; ++i) qlen[i] = q_start[i + 1] - q_start[i];
  const int G = cfg->n_q_heads / cfg->n_kv_heads;
  std::vector<AttnItem> items;
  int n_ws = 0;
  int n_dec = 0;
  std::vector<int> seg_start;
  int n_pf = 0;
  plan_attention(n_seqs, qlen.data(), ctx, cfg->n_kv_heads, G, items, n_ws, n_dec, seg_start, n_pf);
  const int n_cta = seg_start.empty() ? 0 : (int)seg_start.size() - 1;
  alignas(128) uint8_t map[128];
  uint64_t rows = (uint64_t)num_blocks * cfg->n_layers * 2 * cfg->n_kv_heads * block_tokens;
  if (make_kv_tensor_map(map, kv_pool, rows) != 0) return fail(PPD_ERR_CUDA, "tensor map encode failed");
  size_t nb = (size_t)n_seqs * max_blocks;
  size_t bytes = (n_seqs + 1 + n_seqs + nb) * 4 + items.size() * sizeof(AttnItem) + seg_start.size() * 4 + 64;
  uint8_t* dm = nullptr;
  float *ws_o = nullptr, *ws_ml = nullptr;
  int* ctr = nullptr;
  CU(cudaMalloc(&dm, bytes));
  CU(cudaMalloc(&ws_o, (size_t)std::max(n_ws, 1) * cfg->n_kv_heads * G * 128 * 4));
  CU(cudaMalloc(&ws_ml, (size_t)std::max(n_ws, 1) * cfg->n_kv_heads * G * 2 * 4));
  CU(cudaMalloc(&ctr, ((size_t)n_seqs * cfg->n_kv_heads + 4) * 4));
  CU(cudaMemset(ctr, 0, ((size_t)n_seqs * cfg->n_kv_heads + 4) * 4));
  int* d_qs = reinterpret_cast<int*>(dm);
  int* d_ctx = d_qs + n_seqs + 1;
  int* d_bt = d_ctx + n_seqs;
  AttnItem* d_items = reinterpret_cast<AttnItem*>(align_up(reinterpret_cast<uintptr_t>(d_bt + nb), 16));
  CU(cudaMemcpy(d_qs, q_start, (n_seqs + 1) * 4, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(d_ctx, ctx, n_seqs * 4, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(d_bt, block_tables, nb * 4, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(d_items, items.data(), items.size() * sizeof(AttnItem), cudaMemcpyHostToDevice));
  int* d_seg = reinterpret_cast<int*>(d_items + items.size());
  if (!seg_start.empty()) CU(cudaMemcpy(d_seg, seg_start.data(), seg_start.size() * 4, cudaMemcpyHostToDevice));
  rc = run_attention(*cfg, map, static_cast<const bf16*>(q), static_cast<bf16*>(out), d_qs, d_ctx,
                     d_bt, max_blocks, d_items, n_dec, (int)items.size(), d_seg, n_cta, n_pf, layer, ws_o, ws_ml, ctr,
                     ctr + (size_t)n_seqs * cfg->n_kv_heads, s);
  cudaStreamSynchronize(s);
  cudaFree(dm);
  cudaFree(ws_o);
  cudaFree(ws_ml);
  cudaFree(ctr);
  if (rc) return rc;
  CU(cudaGetLastError());
  return PPD_OK;
}

int ppd_op_gemm(const void* A, const void* B, void* C, int32_t M, int32_t N, int32_t K,
                int32_t out_f32, void* stream) {
  CHECK_ARG(A && B && C && M > 0 && N > 0 && K > 0, "bad gemm args");
  static thread_local GemmContext* ctx = nullptr;
  if (!ctx) ctx = gemm_create();
  if (!ctx) return fail(PPD_ERR_CUDA, "gemm context");
  CU(gemm_run_cublas(ctx, static_cast<const bf16*>(A), static_cast<const bf16*>(B), C, M, N, K, out_f32 != 0,
                     static_cast<cudaStream_t>(stream)));
  return PPD_OK;
}

int ppd_op_gemm_tc(const void* A, const void* B, void* C, int32_t M, int32_t N, int32_t K, int32_t out_f32,
                   int32_t splits, void* stream) {
  CHECK_ARG(A && B && C && M > 0 && N > 0 && K > 0 && splits >= 1, "bad gemm args");
  CHECK_ARG(K % 8 == 0, "K must be a multiple of 8");
  CHECK_ARG(splits == 1 || out_f32, "K-split partials need fp32 output");
  CU(gemm_tc_run(static_cast<const bf16*>(A), static_cast<const bf16*>(B), C, M, N, K, out_f32 != 0, splits,
                 (size_t)M * N, static_cast<cudaStream_t>(stream)));
  return PPD_OK;
}

int ppd_op_gemm_silu(const void* A, const void* B, void* m, int32_t M, int32_t N, int32_t K, void* stream) {
  CHECK_ARG(A && B && m && M > 0 && N > 0 && K > 0, "bad gemm args");
  CHECK_ARG(K % 8 == 0 && N % 128 == 0, "K must be a multiple of 8 and N of 128");
  CU(gemm_tc_run_silu(static_cast<const bf16*>(A), static_cast<const bf16*>(B), static_cast<bf16*>(m), M, N, K,
                      static_cast<cudaStream_t>(stream)));
  return PPD_OK;
}

int ppd_op_gemm_parts(const void* A, const void* B, void* C, int32_t M, int32_t N, int32_t K,
                      int32_t max_slices, ppd_gemm_parts* parts, void* stream) {
  CHECK_ARG(A && B && C && parts && M > 0 && N > 0 && K > 0 && max_slices >= 1, "bad gemm args");
  CHECK_ARG(K % 8 == 0, "K must be a multiple of 8");
  GemmParts g;
  CU(gemm_tc_run_parts(static_cast<const bf16*>(A), static_cast<const bf16*>(B), static_cast<float*>(C), M, N, K,
                       max_slices, (size_t)M * N, &g, static_cast<cudaStream_t>(stream)));
  parts->n = g.n;
  parts->kbt = g.kbt;
  parts->slots = g.slots;
  parts->rows = g.rows;
  parts->bn = g.bn;
  parts->n_tiles_t = g.n_tiles_t;
  parts->total = g.total;
  parts->stride = g.stride;
  parts->dp = g.dp;
  return PPD_OK;
}

int ppd_set_tuning(const char* name, int32_t value) {
  static int pair = -1, stages = 0, sched = -1;
  CHECK_ARG(name, "null tuning name");
  if (std::strcmp(name, "gemm_pair") == 0) {
    CHECK_ARG(value >= -1 && value <= 1, "gemm_pair must be -1, 0 or 1");
    pair = value;
  } else if (std::strcmp(name, "gemm_sched") == 0) {
    CHECK_ARG(value >= -1 && value <= 1, "gemm_sched must be -1, 0 or 1");
    sched = value;
  } else if (std::strcmp(name, "gemm_stages") == 0) {
    CHECK_ARG(value >= 0 && value <= 16, "gemm_stages must be in [0, 16]");
    stages = value;
  } else if (std::strcmp(name, "attn_pf_ctas") == 0) {
    CHECK_ARG(value >= 0 && value <= 146, "attn_pf_ctas must be in [0, 146]");
    g_attn_pf_ctas = value;
  } else if (std::strcmp(name, "attn_pf_persist") == 0) {
    CHECK_ARG(value == 0 || value == 1, "attn_pf_persist must be 0 or 1");
    g_attn_pf_persist = value != 0;
  } else if (std::strcmp(name, "attn_fused") == 0) {
    CHECK_ARG(value >= 0 && value <= 2, "attn_fused must be 0, 1 or 2");
    g_attn_fused = value;
  } else if (std::strcmp(name, "gemm_occ2") == 0) {
    CHECK_ARG(value >= -1 && value <= 1, "gemm_occ2 must be -1, 0 or 1");
    gemm_tc_set_occ2(value);
  } else if (std::strcmp(name, "gemm_multi_sub") == 0) {
    CHECK_ARG(value >= 0 && value <= 3, "gemm_multi_sub must be 0, 1, 2 or 3");
    gemm_tc_set_multi_sub(value);
  } else if (std::strcmp(name, "l2_hint") == 0) {
    CHECK_ARG(value >= 0 && value <= 3, "l2_hint must be in [0, 3]");
    gemm_tc_set_l2_hint(value);
  } else if (std::strcmp(name, "gemm_epi_pipe") == 0) {
    CHECK_ARG(value == 0 || value == 1, "gemm_epi_pipe must be 0 or 1");
    gemm_tc_set_epi_pipe(value != 0);
  } else if (std::strcmp(name, "ws_two_slices") == 0) {  // takes effect for devices opened afterwards
    CHECK_ARG(value == 0 || value == 1, "ws_two_slices must be 0 or 1");
    g_ws_two_slices = value != 0;
  } else if (std::strcmp(name, "gemm_even_tiles") == 0) {
    CHECK_ARG(value == 0 || value == 1, "gemm_even_tiles must be 0 or 1");
    gemm_tc_set_even_tiles(value != 0);
  } else if (std::strcmp(name, "pdl_overlap") == 0) {
    CHECK_ARG(value == 0 || value == 1, "pdl_overlap must be 0 or 1");
    set_pdl_overlap(value);
  } else if (std::strcmp(name, "gemm_l2_pre") == 0) {
    CHECK_ARG(value >= -1 && value <= 256, "gemm_l2_pre must be in [-1, 256]");
    gemm_tc_set_l2_pre(value);
  } else if (std::strcmp(name, "layer_kernel") == 0) {
    CHECK_ARG(value == 0 || value == 1, "layer_kernel must be 0 or 1");
    g_layer_kernel = value != 0;
  } else if (std::strcmp(name, "layer_l2_ahead") == 0) {
    CHECK_ARG(value >= 0 && value <= 256, "layer_l2_ahead must be in [0, 256]");
    g_layer_l2_ahead = value;
  } else if (std::strcmp(name, "layer_stages") == 0) {
    CHECK_ARG(value >= 0 && value <= 8, "layer_stages must be in [0, 8]");
    g_layer_stages = value;
  } else if (std::strcmp(name, "mlp_fused") == 0) {
    CHECK_ARG(value >= 0 && value <= 2, "mlp_fused must be 0, 1 or 2");
    g_mlp_fused = value;
  } else {
    return fail(PPD_ERR_INVALID, std::string("unknown tuning knob: ") + name);
  }
  gemm_tc_set_tuning(pair, stages, sched);
  ++g_tuning_epoch;
  return PPD_OK;
}

int ppd_op_fill_random(void* dst, uint64_t n, uint64_t seed, int32_t tensor, int32_t layer,
                       void* stream) {
  CHECK_ARG(dst, "null dst");
  CU(launch_fill_random(static_cast<bf16*>(dst), n, seed, tensor, layer,
                        static_cast<cudaStream_t>(stream)));
  CU(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  return PPD_OK;
}

}  // extern "C"
