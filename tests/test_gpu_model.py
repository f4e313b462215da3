"""End-to-end parity of ppd_step (the fused forward step behind the C-ABI)
against the CPU model oracle on the builder-defined tiny config:
random-init weights from the shared counter hash, paged KV through host block
tables, greedy tokens.

Stated tolerances: logits |gpu - oracle| <= 3e-2 (fp32 logits of magnitude
~0.5; bf16 storage points may round differently after differently-ordered
fp32 accumulation); greedy token ids must be IDENTICAL wherever the oracle's
top-1/top-2 margin exceeds 0.05 (below that an fp32-ulp difference can
legitimately flip the argmax)."""
import numpy as np
import pytest

import paper_2603_13358_b200 as ppd
from oracle import oracle as O

pytestmark = pytest.mark.gpu

LOGIT_ATOL = 3e-2
MARGIN = 0.05
SEED = 20260313


@pytest.fixture(scope="module")
def pair(gpu):
    cfg = ppd.tiny_cfg()
    dev = ppd.Device(0, cfg, max_step_tokens=1024, max_step_seqs=64)
    dev.load_random_weights(SEED)
    dev.kv_pool_init(96)
    model = O.Model(O.cfg_from(cfg), SEED)
    pool = O.KvPool(O.cfg_from(cfg), 96)
    yield cfg, dev, model, pool
    dev.close()


def compare(dev, model, pool, q_len, ctx, tokens, bts):
    r = dev.step(q_len, ctx, tokens, bts)
    logits = dev.last_logits(len(q_len))
    t_o, l_o, margin = model.step(pool, q_len, ctx, tokens, bts)
    assert np.abs(logits - l_o).max() <= LOGIT_ATOL, np.abs(logits - l_o).max()
    sure = margin > MARGIN
    assert (r.tokens[sure] == t_o[sure]).all(), (r.tokens, t_o, margin)
    return r.tokens, t_o


def test_prefill_decode_append_parity(pair):
    cfg, dev, model, pool = pair
    rng = np.random.default_rng(11)
    # two conversations, 8 blocks each
    bts = np.array([np.arange(0, 8), np.arange(8, 16)], dtype=np.int32)
    a = rng.integers(0, cfg.vocab, 37)
    b = rng.integers(0, cfg.vocab, 20)
    tok, _ = compare(dev, model, pool, [37, 20], [0, 0], np.concatenate([a, b]), bts)
    ctx = np.array([37, 20])
    # greedy decode, both rows
    for _ in range(6):
        tok, _ = compare(dev, model, pool, [1, 1], ctx, tok, bts)
        ctx += 1
    # turn 2 of A (append 25 new tokens) rides in the same step as B's decode
    new = rng.integers(0, cfg.vocab, 25)
    tok, _ = compare(dev, model, pool, [25, 1], ctx, np.concatenate([new, tok[1:]]), bts)
    ctx += [25, 1]
    for _ in range(3):
        tok, _ = compare(dev, model, pool, [1, 1], ctx, tok, bts)
        ctx += 1


@pytest.mark.parametrize("knobs", [
    {"gemm_pair": 1, "gemm_sched": 1, "mlp_fused": 1},   # CTA-pair GEMM, balanced partition, fused SiLU
    {"gemm_pair": 0, "gemm_sched": 1, "mlp_fused": 0},   # single-CTA, balanced partition + silu_mul
    {"gemm_pair": 1, "gemm_sched": 0, "mlp_fused": 0},   # CTA-pair, uniform K split
], ids=["pair-balanced-fused", "single-balanced", "pair-uniform"])
def test_step_parity_under_gemm_variants(pair, knobs):
    """Every GEMM schedule / epilogue variant the tuning knobs select keeps the
    forward step at oracle parity (graphs are re-captured on each change)."""
    L = ppd.lib()
    try:
        for k, v in knobs.items():
            ppd.check(L.ppd_set_tuning(k.encode(), v))
        test_prefill_decode_append_parity(pair)
    finally:
        for k, v in (("gemm_pair", -1), ("gemm_sched", -1), ("mlp_fused", 2)):
            ppd.check(L.ppd_set_tuning(k.encode(), v))


def test_kv_pool_contents_match_oracle(pair):
    cfg, dev, model, pool = pair
    import torch
    ptr, nbytes = dev.kv_pool_ptr()
    # copy the device pool back through torch (device pointer -> host)
    host = np.empty(nbytes // 2, dtype=np.uint16)
    import ctypes
    cudart = ctypes.CDLL("libcudart.so")
    cudart.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
    assert cudart.cudaMemcpy(host.ctypes.data, ptr, nbytes, 2) == 0
    got = O.bf16_to_f32(host.reshape(pool.data.shape)[:16])
    want = O.bf16_to_f32(pool.data[:16])
    assert np.abs(got - want).max() <= 2e-2 + 2e-2 * np.abs(want).max()


def test_prefill_seam_full_vs_append(pair):
    """ppd_prefill(FULL) of ctx+new == ppd_prefill(APPEND) of new over ctx
    (the two routes of simulator.cpp:282-311 produce the same next token)."""
    cfg, dev, model, pool = pair
    rng = np.random.default_rng(12)
    hist = rng.integers(0, cfg.vocab, 90)
    bt_full = np.arange(40, 48, dtype=np.int32)
    bt_app = np.arange(48, 56, dtype=np.int32)
    full = dev.prefill(ppd.PREFILL_FULL, hist, 0, bt_full)
    dev.prefill(ppd.PREFILL_FULL, hist[:60], 0, bt_app)
    app = dev.prefill(ppd.PREFILL_APPEND, hist[60:], 60, bt_app)
    lf = None
    t_o, l_o, margin = model.step(O.KvPool(O.cfg_from(cfg), 8), [90], [0], hist, [np.arange(8)])
    if margin[0] > MARGIN:
        assert full.tokens[0] == t_o[0] == app.tokens[0]
    with pytest.raises(ppd.InvalidArgument):
        dev.prefill(ppd.PREFILL_FULL, hist, 5, bt_full)
    with pytest.raises(ppd.InvalidArgument):
        dev.prefill(ppd.PREFILL_APPEND, hist[:0], 5, bt_full)


def test_kv_copy_delta_then_decode(pair):
    """x=0 path on one GPU: P node runs the full prefill, ships the delta
    tokens to D (token-granular, partial first block), D decodes."""
    cfg, dev_d, model, _ = pair
    rng = np.random.default_rng(13)
    dev_p = ppd.Device(0, cfg, max_step_tokens=1024, max_step_seqs=16)
    dev_p.load_random_weights(SEED)
    dev_p.kv_pool_init(32)
    hist = rng.integers(0, cfg.vocab, 70)
    bt_p = np.arange(3, 11, dtype=np.int32)
    bt_d = np.arange(60, 68, dtype=np.int32)
    # D already holds the first 21 positions (from an earlier turn)
    dev_d.prefill(ppd.PREFILL_FULL, hist[:21], 0, bt_d)
    r_p = dev_p.prefill(ppd.PREFILL_FULL, hist, 0, bt_p)
    ms = ppd.kv_copy(dev_p, dev_d, bt_p, bt_d, 21, 70 - 21)
    assert ms >= 0
    # D decodes the P-produced token over the transferred KV; compare to the oracle
    r_d = dev_d.step([1], [70], r_p.tokens, bt_d)
    opool = O.KvPool(O.cfg_from(cfg), 8)
    t1, _, m1 = model.step(opool, [70], [0], hist, [np.arange(8)])
    t2, _, m2 = model.step(opool, [1], [70], t1, [np.arange(8)])
    if m1[0] > MARGIN:
        assert r_p.tokens[0] == t1[0]
    if m1[0] > MARGIN and m2[0] > MARGIN:
        assert r_d.tokens[0] == t2[0]
    dev_p.close()


def test_qwen_shape_bias_group5_parity(gpu):
    """Qwen2.5-style numerics (QKV bias, GQA group 5, theta 1e6, eps 1e-6) on a
    tiny shape: prefill + decode + append through ppd_step vs the oracle."""
    cfg = ppd.ModelCfg(2, 640, 5, 1, 128, 1280, 2048, 1e-6, 1e6, 1)
    dev = ppd.Device(0, cfg, max_step_tokens=512, max_step_seqs=8)
    dev.load_random_weights(77)
    dev.kv_pool_init(32)
    model = O.Model(O.cfg_from(cfg), 77)
    pool = O.KvPool(O.cfg_from(cfg), 32)
    rng = np.random.default_rng(21)
    bts = np.array([np.arange(0, 8), np.arange(8, 16)], dtype=np.int32)
    tok, _ = compare(dev, model, pool, [45, 13], [0, 0], rng.integers(0, cfg.vocab, 58), bts)
    ctx = np.array([45, 13])
    for _ in range(3):
        tok, _ = compare(dev, model, pool, [1, 1], ctx, tok, bts)
        ctx += 1
    new = rng.integers(0, cfg.vocab, 30)
    compare(dev, model, pool, [1, 30], ctx, np.concatenate([tok[:1], new]), bts)
    dev.close()


def test_prefill_size_step_fused_silu_auto(pair):
    """A step of >= 512 token rows takes the default fused-SiLU gate|up GEMM
    (device.cu kMlpFusedMinRows) and, for pure prefill, the persistent tcgen05
    prefill attention: a 600-token full prefill + a 130-token append over it in
    one later step, then decode, all against the oracle."""
    cfg, dev, model, pool = pair
    rng = np.random.default_rng(29)
    bts = np.array([np.arange(16, 56), np.arange(56, 96)], dtype=np.int32)  # 40 blocks = 640 tokens each
    a = rng.integers(0, cfg.vocab, 600)
    tok, _ = compare(dev, model, pool, [600], [0], a, bts[:1])
    b = rng.integers(0, cfg.vocab, 430)
    tok_b, _ = compare(dev, model, pool, [430], [0], b, bts[1:])
    # one 531-row step: A decodes while B appends 130 tokens over its 430
    new = rng.integers(0, cfg.vocab, 130)
    tok2, _ = compare(dev, model, pool, [1, 130], [600, 430], np.concatenate([tok, new]), bts)
    ctx = np.array([601, 560])
    for _ in range(2):
        tok2, _ = compare(dev, model, pool, [1, 1], ctx, tok2, bts)
        ctx += 1
