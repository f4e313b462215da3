"""K1-K4 parity: the sm_100a paged attention (one launch for decode rows and
prefill/append tiles) against the CPU oracle's attention (oracle/model_oracle.c
mo_attention_paged) on identical bf16 q / paged K,V.

Tolerance (stated): |gpu - oracle| <= 2e-2 + 2e-2 * |oracle| elementwise. The
GPU rounds P to bf16 before the PV contraction and stores O in bf16 (the
oracle keeps both fp32), which bounds the error at ~1 bf16 ulp of O plus the
P rounding (2^-9 relative per weight)."""
import numpy as np
import pytest

import paper_2603_13358_b200 as ppd
from oracle import oracle as O

pytestmark = pytest.mark.gpu

ATOL, RTOL = 2e-2, 2e-2


def run_case(cfg, q_len, ctx, seed=0, num_blocks=None, layer=0):
    import torch
    rng = np.random.default_rng(seed)
    n = len(q_len)
    need = [((c + q + 15) // 16) for c, q in zip(ctx, q_len)]
    maxb = max(need)
    nb = num_blocks or sum(need) + 3
    perm = rng.permutation(nb)
    bts = np.zeros((n, maxb), dtype=np.int32)
    k = 0
    for s in range(n):
        bts[s, : need[s]] = perm[k : k + need[s]]
        k += need[s]
    pool = O.f32_to_bf16(rng.standard_normal((nb, cfg.n_layers, 2, cfg.n_kv_heads, 16, 128)).astype(np.float32))
    qs = np.concatenate([[0], np.cumsum(q_len)]).astype(np.int32)
    q = O.f32_to_bf16(rng.standard_normal((qs[-1], cfg.n_q_heads, 128)).astype(np.float32))
    want = O.attention(O.cfg_from(cfg), q, pool, 16, layer, qs, np.array(ctx, np.int32), bts)
    dq = torch.from_numpy(q.view(np.int16)).cuda()
    dpool = torch.from_numpy(pool.view(np.int16)).cuda()
    dout = torch.zeros_like(dq)
    ppd.check(ppd.lib().ppd_op_attention(
        ppd.ctypes.byref(cfg), dq.data_ptr(), dpool.data_ptr(), nb, 16, layer, n,
        ppd._ptr(qs), ppd._ptr(np.array(ctx, np.int32)), ppd._ptr(bts), maxb, dout.data_ptr(), None))
    got = O.bf16_to_f32(dout.cpu().numpy().view(np.uint16))
    err = np.abs(got - want) - (ATOL + RTOL * np.abs(want))
    assert np.isfinite(got).all()
    assert err.max() <= 0, f"max excess {err.max()} at {np.unravel_index(err.argmax(), err.shape)}"
    return got, want


def cfg_of(hq, hkv, layers=2):
    c = ppd.tiny_cfg()
    c.n_q_heads, c.n_kv_heads, c.n_layers = hq, hkv, layers
    return c


def test_decode_rows_ragged(gpu):
    run_case(cfg_of(4, 1), [1] * 6, [0, 1, 15, 16, 63, 1000])


def test_decode_llama_group(gpu):
    run_case(cfg_of(32, 8), [1] * 5, [5, 130, 17, 64, 511], layer=1)


def test_decode_long_context_splits(gpu):
    # one sequence: the builder splits its keys across CTAs (split-KV merge path)
    run_case(cfg_of(32, 8), [1], [9000])
    run_case(cfg_of(4, 1), [1, 1], [20000, 3])


def test_full_prefill(gpu):
    run_case(cfg_of(4, 1), [37], [0])
    run_case(cfg_of(32, 8), [200], [0], seed=3)


def test_append_prefill(gpu):
    run_case(cfg_of(4, 1), [100], [250])
    run_case(cfg_of(32, 8), [17, 64], [1000, 1], seed=4)


def test_mixed_decode_and_append(gpu):
    # prefill work exceeds the decode rows' K/V streaming: the decode kernel
    # then the persistent tcgen05 prefill queue (device.cu mixed_step_fits_k2)
    run_case(cfg_of(32, 8), [1, 1, 50, 1, 130], [700, 3, 400, 64, 0], seed=5)


def test_mixed_small_decode_large_append(gpu):
    """The PPD D node's shape at low load: a few decode rows beside a long
    append over a long cached context (split path), Llama and Qwen groups."""
    run_case(cfg_of(32, 8), [1, 1, 1, 300], [2100, 40, 900, 1700], seed=10)
    run_case(cfg_of(40, 8), [1, 1, 260], [700, 3000, 1200], seed=11)


def test_qwen_group_of_5(gpu):
    run_case(cfg_of(40, 8), [1, 1, 33], [300, 7, 90], seed=6)
    run_case(cfg_of(40, 8), [1], [5000], seed=7)


def test_mixed_many_tiles_per_prefill_cta(gpu):
    """K2 fused launch where the SM split gives each prefill CTA several tiles
    (barriers re-armed per tile) next to a heavy decode batch."""
    q_len = [1] * 64 + [512]
    ctx = [2000 + 7 * i for i in range(64)] + [1500]
    run_case(cfg_of(32, 8), q_len, ctx, seed=8)


def test_mixed_fused_and_split_launches_agree(gpu):
    """The one-launch mixed kernel and the two-launch path (attn_fused = 0)
    both match the oracle on the same mixed batch."""
    L = ppd.lib()
    case = ([1, 1, 1, 96, 1, 40], [900, 33, 4000, 700, 1, 0])
    run_case(cfg_of(32, 8), *case, seed=9)
    ppd.check(L.ppd_set_tuning(b"attn_fused", 0))
    try:
        run_case(cfg_of(32, 8), *case, seed=9)
    finally:
        ppd.check(L.ppd_set_tuning(b"attn_fused", 1))
