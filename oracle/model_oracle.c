/* model_oracle.c — TEST INFRASTRUCTURE ONLY: CPU restatement of the decoder the
 * CUDA path executes. See model_oracle.h for the conventions and for why the
 * parity of this file is "unpinned" against the reference (which has no model:
 * SURVEY.md §0, §8c). The KV bookkeeping it is driven with follows the
 * reference's prefix_cache accounting (simulator.cpp:349-359, :371, :428).
 *
 * Compiled with -ffp-contract=off semantics where it matters (RoPE, RMSNorm
 * scale) so those elementwise steps are bit-identical to the device, which uses
 * __fmul_rn/__fadd_rn there. GEMMs and reductions accumulate in fp32 in a
 * different order than the device: parity for those is tolerance-based.
 */
#include "model_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#pragma GCC optimize("fp-contract=off")

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

uint16_t mo_f32_to_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40u);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

float mo_bf16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static inline float rbf(float f) { return mo_bf16_to_f32(mo_f32_to_bf16(f)); }

uint16_t mo_weight_bf16(uint64_t seed, int tensor, int layer, uint64_t idx) {
  uint64_t key = seed * 0x9E3779B97F4A7C15ULL + ((uint64_t)tensor << 56) +
                 ((uint64_t)layer << 44) + idx;
  uint64_t z = mix64(key);
  float u = (float)(uint32_t)(z >> 40) * 0x1p-24f;
  float v = 2.0f * u - 1.0f;
  float w = v * 0.034641016f;
  return mo_f32_to_bf16(w);
}

uint32_t mo_token_id(uint64_t seed, uint64_t conv_hash, int turn, int64_t pos, int vocab) {
  uint64_t z = mix64(seed ^ mix64(conv_hash + 0x632BE59BD9B4E019ULL * (uint64_t)(turn + 1)) ^
                     (uint64_t)pos * 0xD6E8FEB86659FD93ULL);
  return (uint32_t)(z % (uint64_t)vocab);
}

void mo_rope_table(float theta, int head_dim, int max_pos, float* cos_out, float* sin_out) {
  int half = head_dim / 2;
  for (int p = 0; p < max_pos; ++p)
    for (int i = 0; i < half; ++i) {
      double inv = pow((double)theta, -2.0 * (double)i / (double)head_dim);
      double a = (double)p * inv;
      cos_out[(size_t)p * half + i] = (float)cos(a);
      sin_out[(size_t)p * half + i] = (float)sin(a);
    }
}

/* ------------------------------------------------------------------------ */

typedef struct {
  uint16_t *wq, *wk, *wv, *wo, *wgate, *wup, *wdown; /* [N][K] bf16 */
  float *bq, *bk, *bv;
} mo_layer;

struct mo_model {
  mo_cfg cfg;
  int n_alloc_layers;
  uint64_t seed;
  mo_layer* layers;
  uint16_t* lm_head;
  int rope_len;
  float *rope_cos, *rope_sin;
};

static uint16_t* gen_tensor(uint64_t seed, int tensor, int layer, size_t n) {
  uint16_t* p = (uint16_t*)malloc(n * sizeof(uint16_t));
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < n; ++i) p[i] = mo_weight_bf16(seed, tensor, layer, i);
  return p;
}

/* n consecutive weights of one logical tensor (the fixture generator loads
 * these into the HF reference models, tests/golden/make_hf_fixtures.py) */
void mo_fill_tensor(uint64_t seed, int tensor, int layer, uint64_t n, uint16_t* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)n; ++i) out[i] = mo_weight_bf16(seed, tensor, layer, (uint64_t)i);
}

static float* gen_bias(uint64_t seed, int tensor, int layer, size_t n) {
  float* p = (float*)malloc(n * sizeof(float));
  for (size_t i = 0; i < n; ++i) p[i] = mo_bf16_to_f32(mo_weight_bf16(seed, tensor, layer, i));
  return p;
}

mo_model* mo_model_create(const mo_cfg* cfg, uint64_t seed) {
  mo_model* m = (mo_model*)calloc(1, sizeof(mo_model));
  m->cfg = *cfg;
  m->n_alloc_layers = cfg->n_layers;
  m->seed = seed;
  int L = cfg->n_layers, d = cfg->d_model, Dh = cfg->head_dim;
  size_t qd = (size_t)cfg->n_q_heads * Dh, kd = (size_t)cfg->n_kv_heads * Dh;
  m->layers = (mo_layer*)calloc((size_t)L, sizeof(mo_layer));
  for (int l = 0; l < L; ++l) {
    mo_layer* w = &m->layers[l];
    w->wq = gen_tensor(seed, MO_T_WQ, l, qd * d);
    w->wk = gen_tensor(seed, MO_T_WK, l, kd * d);
    w->wv = gen_tensor(seed, MO_T_WV, l, kd * d);
    w->wo = gen_tensor(seed, MO_T_WO, l, (size_t)d * qd);
    w->wgate = gen_tensor(seed, MO_T_WGATE, l, (size_t)cfg->d_ff * d);
    w->wup = gen_tensor(seed, MO_T_WUP, l, (size_t)cfg->d_ff * d);
    w->wdown = gen_tensor(seed, MO_T_WDOWN, l, (size_t)d * cfg->d_ff);
    if (cfg->qkv_bias) {
      w->bq = gen_bias(seed, MO_T_BQ, l, qd);
      w->bk = gen_bias(seed, MO_T_BK, l, kd);
      w->bv = gen_bias(seed, MO_T_BV, l, kd);
    }
  }
  m->lm_head = gen_tensor(seed, MO_T_LMHEAD, 0, (size_t)cfg->vocab * d);
  m->rope_len = 0;
  return m;
}

/* Runs only the first n layers in mo_step (timing extrapolation in bench.py). */
void mo_set_active_layers(mo_model* m, int n) {
  if (n >= 1 && n <= m->n_alloc_layers) m->cfg.n_layers = n;
}

void mo_model_free(mo_model* m) {
  if (!m) return;
  for (int l = 0; l < m->n_alloc_layers; ++l) {
    mo_layer* w = &m->layers[l];
    free(w->wq); free(w->wk); free(w->wv); free(w->wo);
    free(w->wgate); free(w->wup); free(w->wdown);
    free(w->bq); free(w->bk); free(w->bv);
  }
  free(m->layers);
  free(m->lm_head);
  free(m->rope_cos);
  free(m->rope_sin);
  free(m);
}

static void ensure_rope(mo_model* m, int max_pos) {
  if (max_pos <= m->rope_len) return;
  int n = 1024;
  while (n < max_pos) n *= 2;
  int half = m->cfg.head_dim / 2;
  free(m->rope_cos);
  free(m->rope_sin);
  m->rope_cos = (float*)malloc((size_t)n * half * sizeof(float));
  m->rope_sin = (float*)malloc((size_t)n * half * sizeof(float));
  mo_rope_table(m->cfg.rope_theta, m->cfg.head_dim, n, m->rope_cos, m->rope_sin);
  m->rope_len = n;
}

/* y[r][n] = sum_k x[r][k] * W[n][k]  (fp32 accumulate), W bf16 [N][K]. */
static void gemm_xwT(const float* x, int R, int K, const uint16_t* W, int N, float* y) {
#pragma omp parallel
  {
    float* wbuf = (float*)malloc((size_t)8 * K * sizeof(float));
#pragma omp for schedule(dynamic, 4)
    for (int n0 = 0; n0 < N; n0 += 8) {
      int nb = N - n0 < 8 ? N - n0 : 8;
      for (int j = 0; j < nb; ++j)
        for (int k = 0; k < K; ++k) wbuf[(size_t)j * K + k] = mo_bf16_to_f32(W[(size_t)(n0 + j) * K + k]);
      for (int r = 0; r < R; ++r) {
        const float* xr = x + (size_t)r * K;
        for (int j = 0; j < nb; ++j) {
          const float* wr = wbuf + (size_t)j * K;
          float acc = 0.f;
#pragma omp simd reduction(+ : acc)
          for (int k = 0; k < K; ++k) acc += xr[k] * wr[k];
          y[(size_t)r * N + n0 + j] = acc;
        }
      }
    }
    free(wbuf);
  }
}

static void rmsnorm_rows(const float* x, int R, int d, float eps, float* out) {
#pragma omp parallel for schedule(static)
  for (int r = 0; r < R; ++r) {
    const float* xr = x + (size_t)r * d;
    float ss = 0.f;
    for (int i = 0; i < d; ++i) ss += xr[i] * xr[i];
    float inv = 1.0f / sqrtf(ss / (float)d + eps);
    for (int i = 0; i < d; ++i) out[(size_t)r * d + i] = rbf(xr[i] * inv); /* norm weight = 1 */
  }
}

static inline size_t kv_index(const mo_cfg* c, int block_tokens, int blk, int layer, int kv, int h,
                              int t, int dim) {
  return (((((size_t)blk * c->n_layers + layer) * 2 + kv) * c->n_kv_heads + h) * block_tokens + t) *
             c->head_dim + dim;
}

void mo_attention_paged(const mo_cfg* c, const uint16_t* q, const uint16_t* kv, int bt, int layer,
                        int n_seqs, const int32_t* q_start, const int32_t* ctx,
                        const int32_t* block_tables, int max_blocks, float* out) {
  int Hq = c->n_q_heads, Hkv = c->n_kv_heads, Dh = c->head_dim, grp = Hq / Hkv;
  int total_q = q_start[n_seqs];
  float scale = 1.0f / sqrtf((float)Dh);
#pragma omp parallel
  {
    int cap = 0;
    float* sc = NULL;
#pragma omp for schedule(dynamic, 1) collapse(2)
    for (int row = 0; row < total_q; ++row)
      for (int h = 0; h < Hq; ++h) {
        int s = 0;
        while (q_start[s + 1] <= row) ++s;
        int pos = ctx[s] + (row - q_start[s]);
        int nk = pos + 1;
        if (nk > cap) {
          cap = nk * 2;
          sc = (float*)realloc(sc, (size_t)cap * sizeof(float));
        }
        const uint16_t* qr = q + ((size_t)row * Hq + h) * Dh;
        int hk = h / grp;
        float mx = -INFINITY;
        for (int j = 0; j < nk; ++j) {
          int blk = block_tables[(size_t)s * max_blocks + j / bt];
          const uint16_t* kr = kv + kv_index(c, bt, blk, layer, 0, hk, j % bt, 0);
          float acc = 0.f;
#pragma omp simd reduction(+ : acc)
          for (int d = 0; d < Dh; ++d) acc += mo_bf16_to_f32(qr[d]) * mo_bf16_to_f32(kr[d]);
          sc[j] = acc * scale;
          if (sc[j] > mx) mx = sc[j];
        }
        float sum = 0.f;
        for (int j = 0; j < nk; ++j) {
          sc[j] = expf(sc[j] - mx);
          sum += sc[j];
        }
        float* o = out + ((size_t)row * Hq + h) * Dh;
        for (int d = 0; d < Dh; ++d) o[d] = 0.f;
        for (int j = 0; j < nk; ++j) {
          int blk = block_tables[(size_t)s * max_blocks + j / bt];
          const uint16_t* vr = kv + kv_index(c, bt, blk, layer, 1, hk, j % bt, 0);
          float p = sc[j];
          for (int d = 0; d < Dh; ++d) o[d] += p * mo_bf16_to_f32(vr[d]);
        }
        float inv = 1.0f / sum;
        for (int d = 0; d < Dh; ++d) o[d] *= inv;
      }
    free(sc);
  }
}

static void rope_rows(const mo_model* m, float* x, int R, int n_heads, const int32_t* pos) {
  int Dh = m->cfg.head_dim, half = Dh / 2;
  for (int r = 0; r < R; ++r)
    for (int h = 0; h < n_heads; ++h) {
      float* v = x + ((size_t)r * n_heads + h) * Dh;
      const float* cs = m->rope_cos + (size_t)pos[r] * half;
      const float* sn = m->rope_sin + (size_t)pos[r] * half;
      for (int i = 0; i < half; ++i) {
        float x1 = v[i], x2 = v[i + half];
        float a = x1 * cs[i];
        float b = x2 * sn[i];
        float c2 = x2 * cs[i];
        float d2 = x1 * sn[i];
        v[i] = rbf(a - b);
        v[i + half] = rbf(c2 + d2);
      }
    }
}

int mo_step(mo_model* m, uint16_t* kv, int bt, int n_seqs, const int32_t* q_start,
            const int32_t* ctx, const int32_t* tokens, const int32_t* block_tables, int max_blocks,
            float* logits_out, int32_t* tokens_out, float* margin_out) {
  const mo_cfg* c = &m->cfg;
  int R = q_start[n_seqs];
  int d = c->d_model, Dh = c->head_dim, Hq = c->n_q_heads, Hkv = c->n_kv_heads, F = c->d_ff;
  int qd = Hq * Dh, kd = Hkv * Dh;
  int32_t* pos = (int32_t*)malloc((size_t)R * sizeof(int32_t));
  int maxpos = 1;
  for (int s = 0; s < n_seqs; ++s)
    for (int r = q_start[s]; r < q_start[s + 1]; ++r) {
      pos[r] = ctx[s] + (r - q_start[s]);
      if (pos[r] + 1 > maxpos) maxpos = pos[r] + 1;
    }
  ensure_rope(m, maxpos);

  float* x = (float*)malloc((size_t)R * d * sizeof(float));
  float* h = (float*)malloc((size_t)R * d * sizeof(float));
  float* qb = (float*)malloc((size_t)R * qd * sizeof(float));
  float* kb = (float*)malloc((size_t)R * kd * sizeof(float));
  float* vb = (float*)malloc((size_t)R * kd * sizeof(float));
  uint16_t* q16 = (uint16_t*)malloc((size_t)R * qd * sizeof(uint16_t));
  float* att = (float*)malloc((size_t)R * qd * sizeof(float));
  float* g = (float*)malloc((size_t)R * F * sizeof(float));
  float* u = (float*)malloc((size_t)R * F * sizeof(float));
  float* tmp = (float*)malloc((size_t)R * d * sizeof(float));

  for (int r = 0; r < R; ++r)
    for (int i = 0; i < d; ++i)
      x[(size_t)r * d + i] = mo_bf16_to_f32(mo_weight_bf16(m->seed, MO_T_EMBED, 0, (size_t)tokens[r] * d + i));

  for (int l = 0; l < c->n_layers; ++l) {
    const mo_layer* w = &m->layers[l];
    rmsnorm_rows(x, R, d, c->rms_eps, h);
    gemm_xwT(h, R, d, w->wq, qd, qb);
    gemm_xwT(h, R, d, w->wk, kd, kb);
    gemm_xwT(h, R, d, w->wv, kd, vb);
    for (int r = 0; r < R; ++r) {
      for (int i = 0; i < qd; ++i) qb[(size_t)r * qd + i] = rbf(qb[(size_t)r * qd + i] + (w->bq ? w->bq[i] : 0.f));
      for (int i = 0; i < kd; ++i) {
        kb[(size_t)r * kd + i] = rbf(kb[(size_t)r * kd + i] + (w->bk ? w->bk[i] : 0.f));
        vb[(size_t)r * kd + i] = rbf(vb[(size_t)r * kd + i] + (w->bv ? w->bv[i] : 0.f));
      }
    }
    rope_rows(m, qb, R, Hq, pos);
    rope_rows(m, kb, R, Hkv, pos);
    /* write K/V of the new tokens into the pool */
    for (int s = 0; s < n_seqs; ++s)
      for (int r = q_start[s]; r < q_start[s + 1]; ++r) {
        int p = pos[r];
        int blk = block_tables[(size_t)s * max_blocks + p / bt];
        for (int hk = 0; hk < Hkv; ++hk)
          for (int dd = 0; dd < Dh; ++dd) {
            kv[kv_index(c, bt, blk, l, 0, hk, p % bt, dd)] = mo_f32_to_bf16(kb[(size_t)r * kd + hk * Dh + dd]);
            kv[kv_index(c, bt, blk, l, 1, hk, p % bt, dd)] = mo_f32_to_bf16(vb[(size_t)r * kd + hk * Dh + dd]);
          }
      }
    for (size_t i = 0; i < (size_t)R * qd; ++i) q16[i] = mo_f32_to_bf16(qb[i]);
    mo_attention_paged(c, q16, kv, bt, l, n_seqs, q_start, ctx, block_tables, max_blocks, att);
    for (size_t i = 0; i < (size_t)R * qd; ++i) att[i] = rbf(att[i]);
    gemm_xwT(att, R, qd, w->wo, d, tmp);
    for (size_t i = 0; i < (size_t)R * d; ++i) x[i] = rbf(x[i] + rbf(tmp[i]));
    rmsnorm_rows(x, R, d, c->rms_eps, h);
    gemm_xwT(h, R, d, w->wgate, F, g);
    gemm_xwT(h, R, d, w->wup, F, u);
    for (size_t i = 0; i < (size_t)R * F; ++i) {
      float gv = g[i];
      float sv = gv / (1.0f + expf(-gv));
      g[i] = rbf(sv * u[i]);
    }
    gemm_xwT(g, R, F, w->wdown, d, tmp);
    for (size_t i = 0; i < (size_t)R * d; ++i) x[i] = rbf(x[i] + rbf(tmp[i]));
  }

  /* final norm + lm_head on the last row of every sequence */
  float* last = (float*)malloc((size_t)n_seqs * d * sizeof(float));
  float* hl = (float*)malloc((size_t)n_seqs * d * sizeof(float));
  for (int s = 0; s < n_seqs; ++s)
    memcpy(last + (size_t)s * d, x + (size_t)(q_start[s + 1] - 1) * d, (size_t)d * sizeof(float));
  rmsnorm_rows(last, n_seqs, d, c->rms_eps, hl);
  float* logits = (float*)malloc((size_t)n_seqs * c->vocab * sizeof(float));
  gemm_xwT(hl, n_seqs, d, m->lm_head, c->vocab, logits);
  for (int s = 0; s < n_seqs; ++s) {
    const float* lg = logits + (size_t)s * c->vocab;
    int best = 0;
    float b1 = lg[0], b2 = -INFINITY;
    for (int v = 1; v < c->vocab; ++v) {
      if (lg[v] > b1) {
        b2 = b1;
        b1 = lg[v];
        best = v;
      } else if (lg[v] > b2) {
        b2 = lg[v];
      }
    }
    if (tokens_out) tokens_out[s] = best;
    if (margin_out) margin_out[s] = b1 - b2;
  }
  if (logits_out) memcpy(logits_out, logits, (size_t)n_seqs * c->vocab * sizeof(float));

  free(pos); free(x); free(h); free(qb); free(kb); free(vb); free(q16); free(att);
  free(g); free(u); free(tmp); free(last); free(hl); free(logits);
  return 0;
}
