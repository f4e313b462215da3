"""Two-GPU paths (skipped below 2 GPUs; the driver's round-end box and the
8-GPU scaling box exercise them): the P->D KV hop between pools on different
GPUs (peer pointers over NVLink), synchronous and asynchronous, checked
bit-exactly against the source pool and, after the hop, against the CPU
oracle; the real-time engine with one node per GPU; the NVLink probe."""
import numpy as np
import pytest

import paper_2603_13358_b200 as ppd
from paper_2603_13358_b200 import engine as E
from oracle import oracle as O

pytestmark = pytest.mark.gpu
MARGIN = 0.05
SEED = 20260313


def n_gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


needs2 = pytest.mark.skipif(n_gpus() < 2, reason="needs 2 GPUs")


@pytest.mark.parametrize("pair", [(0, 0), pytest.param((0, 1), marks=needs2)], ids=["same-gpu", "gpu0-gpu1"])
def test_kv_hop_async_bit_exact_then_decode(gpu, pair):
    cfg = ppd.tiny_cfg()
    p = ppd.Device(pair[0], cfg, max_step_tokens=1024, max_step_seqs=8)
    d = ppd.Device(pair[1], cfg, max_step_tokens=1024, max_step_seqs=8)
    try:
        for dev in (p, d):
            dev.load_random_weights(SEED)
            dev.kv_pool_init(32)
        rng = np.random.default_rng(13)
        hist = rng.integers(0, cfg.vocab, 70)
        bt_p = np.arange(3, 11, dtype=np.int32)
        bt_d = np.arange(20, 28, dtype=np.int32)
        d.prefill(ppd.PREFILL_FULL, hist[:21], 0, bt_d)      # D holds 21 positions already
        r_p = p.prefill(ppd.PREFILL_FULL, hist, 0, bt_p)      # P recomputes all 70
        t = ppd.kv_copy_submit(p, d, bt_p, bt_d, 21, 70 - 21)  # asynchronous hop of the delta
        assert ppd.kv_copy_wait(d, t) >= 0
        src = p.kv_pool_read().reshape(32, -1)
        dst = d.kv_pool_read().reshape(32, -1)
        shape = (cfg.n_layers, 2, cfg.n_kv_heads, 16, cfg.head_dim)
        for pos in range(21, 70):
            s_blk = src[bt_p[pos // 16]].reshape(shape)[:, :, :, pos % 16]
            d_blk = dst[bt_d[pos // 16]].reshape(shape)[:, :, :, pos % 16]
            assert np.array_equal(s_blk, d_blk), pos
        r_d = d.step([1], [70], r_p.tokens, bt_d)
        model = O.Model(O.cfg_from(cfg), SEED)
        opool = O.KvPool(O.cfg_from(cfg), 8)
        t1, _, m1 = model.step(opool, [70], [0], hist, [np.arange(8)])
        t2, _, m2 = model.step(opool, [1], [70], t1, [np.arange(8)])
        if m1[0] > MARGIN:
            assert r_p.tokens[0] == t1[0]
        if m1[0] > MARGIN and m2[0] > MARGIN:
            assert r_d.tokens[0] == t2[0]
    finally:
        p.close()
        d.close()


@needs2
def test_nvlink_probe_and_k7_between_gpus(gpu):
    assert ppd.p2p_bandwidth(0, 1, 256 << 20, 3, 0) > 50.0
    assert ppd.p2p_bandwidth(0, 1, 256 << 20, 3, 1) > 50.0


@needs2
@pytest.mark.parametrize("x", [0.0, 1.0])
def test_realtime_engine_one_node_per_gpu(gpu, x):
    convs = [{"conv_id": f"c{i}", "arrival": 0.01 * i, "turns": [[40, 6], [24, 5], [17, 4]]} for i in range(4)]
    job = {"cluster": "1P_1D", "x": x, "clock": "realtime", "conversations": convs,
           "device": {"model": "tiny", "weight_seed": 5, "token_seed": 9, "gpus": [0, 1],
                      "prefill_chunk": 32, "record_steps": True}}
    r = E.run(job)
    recs = E.records(r)
    assert len(recs) == 12 and all(v["status"] == "completed" for v in recs)
    assert [n["gpu"] for n in r["device"]["nodes"]] == [0, 1]
    log = r["device"]["step_log"]
    cfg = O.cfg_from(ppd.tiny_cfg())
    model = O.Model(cfg, 5)
    nblocks = max(max(e.get("block_tables", [0]) + e.get("src_blocks", [0]) + e.get("dst_blocks", [0]))
                  for e in log) + 1
    pools = {}
    checked = 0
    for e in log:
        if e.get("copy"):
            src = pools.setdefault(e["src"], O.KvPool(cfg, nblocks)).data
            dst = pools.setdefault(e["dst"], O.KvPool(cfg, nblocks)).data
            for q in range(e["start"], e["start"] + e["n"]):
                dst[e["dst_blocks"][q // 16], :, :, :, q % 16] = src[e["src_blocks"][q // 16], :, :, :, q % 16]
            continue
        pool = pools.setdefault(e["node"], O.KvPool(cfg, nblocks))
        n = len(e["q_len"])
        bt = np.array(e["block_tables"], dtype=np.int32).reshape(n, e["max_blocks"])
        t_o, _, margin = model.step(pool, e["q_len"], e["ctx"], e["tokens"], bt, want_logits=False)
        for i in range(n):
            if e["want"][i] and margin[i] > MARGIN:
                assert e["out"][i] == t_o[i]
                checked += 1
    assert checked > 10
