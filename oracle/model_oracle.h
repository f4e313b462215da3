/* model_oracle.h — TEST INFRASTRUCTURE ONLY (the CPU numerics oracle).
 *
 * parity unpinned: the reference (/root/reference/proj) contains no model, no
 * tensors and no attention. Its execute path is four
 * analytic cost functions (costmodel.cpp:318-379). This file restates the
 * standard Llama-3 / Qwen2.5 decoder that BASELINE.json names, with the
 * builder-defined conventions below; the CUDA path must match it. Only tests,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 *
 * Conventions (shared with the device library, documented in DESIGN.md §3):
 *  - weights: bf16, value = bf16(U(-a, a)), a = 0.02*sqrt(3) (std 0.02), drawn
 *    from a counter hash of (seed, tensor, layer, logical index); norms = 1.
 *  - activations stored bf16 at: embed, norm out, q/k/v, rope out, attn out,
 *    o-proj out, residual, silu(g)*u, down out; logits fp32.
 *  - RMSNorm eps 1e-5; RoPE NeoX (rotate-half) with a host-built double→fp32
 *    cos/sin table; softmax scale 1/sqrt(head_dim); greedy argmax, lowest
 *    index wins ties.
 *  - paged KV pool layout, block-major: [block][layer][K|V][kv_head][tok][dim].
 */
#ifndef PPD_MODEL_ORACLE_H
#define PPD_MODEL_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct mo_cfg {
  int n_layers, d_model, n_q_heads, n_kv_heads, head_dim, d_ff, vocab;
  float rms_eps, rope_theta;
  int qkv_bias;
} mo_cfg;

/* logical tensor ids used by the weight hash */
enum { MO_T_EMBED = 0, MO_T_WQ = 1, MO_T_WK = 2, MO_T_WV = 3, MO_T_WO = 4,
       MO_T_WGATE = 5, MO_T_WUP = 6, MO_T_WDOWN = 7, MO_T_LMHEAD = 8,
       MO_T_BQ = 9, MO_T_BK = 10, MO_T_BV = 11 };

uint16_t mo_weight_bf16(uint64_t seed, int tensor, int layer, uint64_t idx);
uint16_t mo_f32_to_bf16(float f);
/* out[i] = mo_weight_bf16(seed, tensor, layer, i), i < n (OpenMP) */
void mo_fill_tensor(uint64_t seed, int tensor, int layer, uint64_t n, uint16_t* out);
float mo_bf16_to_f32(uint16_t h);
uint32_t mo_token_id(uint64_t seed, uint64_t conv_hash, int turn, int64_t pos, int vocab);

/* cos/sin table [max_pos][head_dim/2] fp32, built in double. */
void mo_rope_table(float theta, int head_dim, int max_pos, float* cos_out, float* sin_out);

typedef struct mo_model mo_model;
mo_model* mo_model_create(const mo_cfg* cfg, uint64_t seed);
void mo_model_free(mo_model* m);
void mo_set_active_layers(mo_model* m, int n);

/* Paged KV pool, bf16, layout above. Caller owns the memory:
 * num_blocks * n_layers * 2 * n_kv_heads * block_tokens * head_dim uint16. */
int mo_step(mo_model* m, uint16_t* kv_pool, int block_tokens,
            int n_seqs, const int32_t* q_start, const int32_t* ctx,
            const int32_t* tokens, const int32_t* block_tables, int max_blocks,
            float* logits_out /* n_seqs*vocab or NULL */,
            int32_t* tokens_out /* n_seqs */, float* margin_out /* n_seqs or NULL */);

/* Attention over the paged pool for one layer, queries already roped (bf16).
 * q: [total_q][n_q_heads][head_dim] bf16; out: same shape, fp32 (unrounded).
 * Query i of sequence s sits at position ctx[s] + i and attends keys
 * 0..ctx[s]+i (causal). Keys/values for all those positions must be in the pool. */
void mo_attention_paged(const mo_cfg* cfg, const uint16_t* q, const uint16_t* kv_pool,
                        int block_tokens, int layer, int n_seqs, const int32_t* q_start,
                        const int32_t* ctx, const int32_t* block_tables, int max_blocks,
                        float* out);

#ifdef __cplusplus
}
#endif
#endif
