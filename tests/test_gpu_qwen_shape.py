"""End-to-end parity of ppd_step at the Qwen2.5-32B SHAPE (BASELINE configs[4]:
d 5120, 40 q / 8 kv heads (GQA group 5), F 27648, V 152064, QKV bias, RoPE
theta 1e6, RMSNorm eps 1e-6; 2 layers so the CPU oracle finishes in seconds)
against the CPU model oracle — pinned to HF transformers' Qwen2ForCausalLM on
the tiny Qwen shape (tests/test_oracle.py) — at the configs[4] step shapes:

* B=16 decode over long cached contexts (the agentic trace's decode batch);
* a 1536-token append over 8192 cached tokens (an agentic turn-2+ append);
* a mixed step: 3 decode rows + a 1024-token append over 6000 cached.

Cached contexts hold random bf16 K/V written identically into the device pool
and the oracle's pool. Tolerance as tests/test_gpu_llama_shape.py."""
import numpy as np
import pytest

import paper_2603_13358_b200 as ppd
from oracle import oracle as O

pytestmark = pytest.mark.gpu

LOGIT_REL = 1.5e-2
MARGIN = 0.05
SEED = 20260317
NB = 3000  # 2 layers x 8 kv heads: 128 KiB per block; disjoint regions per test


@pytest.fixture(scope="module")
def qwen2(gpu):
    cfg = ppd.qwen32b_cfg(n_layers=2)
    dev = ppd.Device(0, cfg, max_step_tokens=4096, max_step_seqs=64)
    dev.load_random_weights(SEED)
    dev.kv_pool_init(NB)
    ocfg = O.cfg_from(cfg)
    model = O.Model(ocfg, SEED)
    pool = O.KvPool(ocfg, NB)
    rng = np.random.default_rng(17)
    pool.data[...] = O.f32_to_bf16(rng.standard_normal(pool.data.shape, dtype=np.float32))
    dev.kv_pool_write(pool.data)
    yield cfg, dev, model, pool
    dev.close()


def compare(dev, model, pool, q_len, ctx, tokens, bts):
    r = dev.step(q_len, ctx, tokens, bts)
    logits = dev.last_logits(len(q_len))
    t_o, l_o, margin = model.step(pool, q_len, ctx, tokens, bts)
    assert np.isfinite(logits).all()
    err = np.abs(logits - l_o).max(axis=1)
    lim = LOGIT_REL * np.abs(l_o).max(axis=1)
    assert (err <= lim).all(), (err, lim)
    sure = margin > MARGIN
    assert (r.tokens[sure] == t_o[sure]).all(), (r.tokens, t_o, margin)
    return r, t_o


def test_decode_b16_long_context(qwen2):
    cfg, dev, model, pool = qwen2
    B, nbk = 16, 100
    bts = np.arange(B * nbk, dtype=np.int32).reshape(B, nbk)
    rng = np.random.default_rng(1)
    tok = rng.integers(0, cfg.vocab, B).astype(np.int32)
    ctx = rng.integers(1000, 1580, B).astype(np.int32)
    for _ in range(2):
        _, tok = compare(dev, model, pool, [1] * B, ctx, tok, bts)
        ctx = ctx + 1


def test_append_1536_over_8192(qwen2):
    cfg, dev, model, pool = qwen2
    bts = np.arange(1600, 1600 + 610, dtype=np.int32)[None]  # 9760 tokens
    toks = np.random.default_rng(2).integers(0, cfg.vocab, 1536).astype(np.int32)
    r, t = compare(dev, model, pool, [1536], [8192], toks, bts)
    compare(dev, model, pool, [1], [8192 + 1536], t, bts)


def test_mixed_3_decode_plus_append_1024_over_6000(qwen2):
    cfg, dev, model, pool = qwen2
    bt = np.zeros((4, 440), dtype=np.int32)
    for i in range(3):
        bt[i, :100] = np.arange(2210 + i * 100, 2210 + (i + 1) * 100)
    bt[3, :440] = np.arange(2510, 2950)                   # 6000 cached + 1024 appended = 7024 tokens
    rng = np.random.default_rng(3)
    toks = rng.integers(0, cfg.vocab, 3 + 1024).astype(np.int32)
    compare(dev, model, pool, [1, 1, 1, 1024], [1200, 900, 1500, 6000], toks, bt)
