"""Device clock: the host C++ engine drives real B200 execution (tiny model).

* transfer accounting on the device equals the reference's rule (delta only,
  simulator.cpp:349-353): x=1 ships only Turn-1 KV, x=0 ships every turn's
  new tokens; byte counts use the device pool's real bytes/token;
* every request emits exactly its target tokens; turn-2+ runs append locally
  under x=1;
* generated token ids are IDENTICAL to the CPU oracle replaying the engine's
  own step log (teacher-forced per step; margin-filtered as in test_gpu_model),
  including steps that read KV shipped P -> D by ppd_kv_copy."""
import numpy as np
import pytest

import paper_2603_13358_b200 as ppd
from paper_2603_13358_b200 import engine as E
from oracle import oracle as O

pytestmark = pytest.mark.gpu
MARGIN = 0.05


def trace(n=3, turns=((40, 6), (24, 5), (17, 4))):
    return [{"conv_id": f"c{i}", "arrival": 0.01 * i, "turns": [list(t) for t in turns]} for i in range(n)]


def dev_job(cluster, x, record_steps=False, **kw):
    return {"cluster": cluster, "x": x, "clock": "device", "conversations": trace(**kw),
            "device": {"model": "tiny", "weight_seed": 5, "token_seed": 9, "gpus": [0],
                       "prefill_chunk": 32, "p_prefill_chunk": 48, "record_steps": record_steps}}


def test_device_replica_completes(gpu):
    r = E.run(dev_job("1R", 0.0))
    recs = E.records(r)
    assert len(recs) == 9 and all(x["status"] == "completed" for x in recs)
    want = {1: 6, 2: 5, 3: 4}
    assert all(x["output_tokens_emitted"] == want[x["turn_index"]] for x in recs)
    toks = r["device"]["tokens"]
    assert all(len(toks[c][str(t)]) == want[t] for c in toks for t in (1, 2, 3))
    assert all(x["route"] == "R_local" for x in recs)


def test_device_transfer_accounting_matches_reference_rule(gpu):
    kvb = ppd.kv_block_bytes(ppd.tiny_cfg()) / 16
    x1 = E.run(dev_job("1P_1D", 1.0))
    x0 = E.run(dev_job("1P_1D", 0.0))
    assert x1["link_transfers"] == 3 and x1["link_bytes"] == 3 * 40 * kvb
    assert x0["link_transfers"] == 9 and x0["link_bytes"] == 3 * (40 + 24 + 17) * kvb
    # identical to the reference's accounting on the same trace (virtual clock, same bytes/token)
    from paper_2603_13358_b200 import engine
    v0 = engine.run({"cluster": "1P_1D", "x": 0.0, "conversations": trace(),
                     "calib_overrides": {"kv_bytes_per_token": kvb}})
    assert v0["link_transfers"] == x0["link_transfers"] and v0["link_bytes"] == x0["link_bytes"]
    r1 = E.records(x1)
    assert [x["route"] for x in r1 if x["turn_index"] > 1] == ["D_local"] * 6
    # PPD appends only the new tokens on D (a pending completion flush is not an eviction)
    d_node = x1["device"]["nodes"][1]
    assert d_node["prefill_tokens"] == 3 * (24 + 17) and d_node["evictions"] == 0
    assert x1["device"]["kv_transfer"]["gbs"] > 0


def test_device_tokens_match_oracle_replay(gpu):
    r = E.run(dev_job("1P_1D", 0.5, record_steps=True))
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
            for p in range(e["start"], e["start"] + e["n"]):
                dst[e["dst_blocks"][p // 16], :, :, :, p % 16] = src[e["src_blocks"][p // 16], :, :, :, p % 16]
            continue
        pool = pools.setdefault(e["node"], O.KvPool(cfg, nblocks))
        n = len(e["q_len"])
        bt = np.array(e["block_tables"], dtype=np.int32).reshape(n, e["max_blocks"])
        t_o, _, margin = model.step(pool, e["q_len"], e["ctx"], e["tokens"], bt, want_logits=False)
        for i in range(n):
            if e["want"][i] and margin[i] > MARGIN:
                assert e["out"][i] == t_o[i], (e["node"], i, e["out"][i], t_o[i], margin[i])
                checked += 1
    assert checked > 20


def test_device_timeouts_and_hybrid(gpu):
    """Timeouts free the batch slot on the device clock too (simulator.cpp:436-445),
    and hybrid R/P/D clusters keep replica-pinned conversations local."""
    job = dev_job("1P_1D", 0.0)
    job["request_timeout_s"] = 1e-4  # every request expires before its first token
    r = E.run(job)
    recs = E.records(r)
    assert len(recs) == 3 and all(x["status"] == "timed_out" for x in recs)
    h = E.run(dev_job("1R_1P_1D", 1.0, n=4))
    routes = {}
    for x in E.records(h):
        routes.setdefault(x["conv_id"], []).append(x["route"])
    for rs in routes.values():
        if rs[0] == "R_local":
            assert all(v == "R_local" for v in rs)
        else:
            assert "R_local" not in rs
    assert all(x["status"] == "completed" for x in E.records(h))


def test_device_clock_sweep_manifest_readable_by_reference(gpu, tmp_path):
    """§8f-2 on real runs: a sweep plan whose every cell executes on the GPU
    (engine device clock). Cells complete, the CSV has one row per cell, and
    the manifest directory is read back unchanged by the reference's own
    run_sweep (it resumes from our cells instead of simulating them)."""
    wl = {"id": "tiny_bal", "turn1": {"input_tokens": 48, "output_tokens": 6},
          "turn2plus": {"input_tokens": 24, "output_tokens": 6}, "num_turns": 2, "qps": 1.0,
          "duration_s": 1.5, "think_time_s": 0.0, "jitter_pct": 0.0}
    plan = {"schema_version": 1,
            "configs": [{"shape": "1P_1D", "x_mode": "x0"}, {"shape": "1P_1D", "x_mode": "x1"},
                        {"shape": "2R", "x_mode": "replica"}],
            "workloads": [wl], "qps_levels": [2.0], "seeds": [1], "duration_s": 1.5}
    job = {"op": "sweep", "plan": plan, "clock": "device", "manifest_dir": str(tmp_path),
           "device": {"model": "tiny", "weight_seed": 5, "token_seed": 9, "gpus": [0], "prefill_chunk": 64},
           "compare": [["x0", "x1", "ttft_t2_mean"]]}
    r = E.run(job)
    assert len(r["cells"]) == 3 and not any(c["failed"] for c in r["cells"])
    assert all(c["metrics"]["success_rate"] == 1.0 for c in r["cells"])
    assert r["csv"].count("\n") == 4
    assert "render" in r["winner"]
    ref = O.ref_tool({"op": "sweep", "plan": plan, "manifest_dir": str(tmp_path)})
    assert ref["cells"] == r["cells"] and ref["csv"] == r["csv"] and ref["winner"] == r["winner"]
    # the virtual clock disagrees with the device clock on these numbers
    virt = E.run({"op": "sweep", "plan": plan})
    assert virt["cells"] != r["cells"]


def test_device_clock_trace_replay(gpu):
    """§8f-4 on the device: a JSONL trace (ingest_trace filters) replayed at a
    fixed QPS through the engine's device clock; every request completes with
    exactly its target output and the routes follow x (x=1: turn 2+ local)."""
    import json as _json
    rng = np.random.default_rng(3)
    lines = []
    for i in range(8):
        turns = [{"input_tokens": int(rng.integers(8, 64)), "output_tokens": int(rng.integers(2, 7))}
                 for _ in range(int(rng.integers(1, 4)))]
        lines.append(_json.dumps({"conv_id": f"t{i}", "turns": turns}))
    job = {"cluster": "1P_1D", "x": 1.0, "clock": "device", "trace_jsonl": "\n".join(lines) + "\n",
           "min_turns": 2, "qps_replay": 4.0, "seed": 2,
           "device": {"model": "tiny", "weight_seed": 5, "token_seed": 9, "gpus": [0], "prefill_chunk": 64}}
    r = E.run(job)
    recs = E.records(r)
    kept = E.run({"op": "ingest_trace", "trace_jsonl": job["trace_jsonl"], "min_turns": 2})["conversations"]
    assert len(recs) == sum(len(c["turns"]) for c in kept) > 0
    want = {(c["conv_id"], i + 1): t[1] for c in kept for i, t in enumerate(c["turns"])}
    assert all(x["status"] == "completed" and x["output_tokens_emitted"] == want[(x["conv_id"], x["turn_index"])]
               for x in recs)
    assert all(x["route"] == "D_local" for x in recs if x["turn_index"] > 1)


@pytest.mark.parametrize("cluster", ["2P_6D", "4P_4D"])
@pytest.mark.parametrize("x", [0.0, 1.0])
def test_device_eight_node_layouts(gpu, cluster, x):
    """configs[3]-shaped multi-turn load on the 8-node layouts, all nodes on
    one GPU (tiny model): every request completes with its target tokens and
    the link carries the reference's delta rule."""
    wl = {"id": "cfg4_tiny", "turn1": [64, 6], "turn2plus": [32, 6], "num_turns": 3, "qps": 24.0, "duration_s": 1.0}
    job = {"cluster": cluster, "x": x, "clock": "device", "seed": 3, "workload": wl,
           "device": {"model": "tiny", "weight_seed": 5, "token_seed": 9, "gpus": [0], "prefill_chunk": 64}}
    r = E.run(job)
    recs = E.records(r)
    assert recs and all(x_["status"] == "completed" for x_ in recs)
    assert all(x_["output_tokens_emitted"] == 6 for x_ in recs)
    ref = E.run(dict(job, clock="virtual"))
    assert len(E.records(ref)) == len(recs)


def rt_job(cluster, x, **kw):
    j = dev_job(cluster, x, **kw)
    j["clock"] = "realtime"
    return j


@pytest.mark.parametrize("x", [0.0, 0.5, 1.0])
def test_kv_pool_lifecycle_small_pool(gpu, x):
    """Conversation tables are released at their last turn, admission control
    waits for room instead of aborting ("KV pool exhausted" in round 1): a
    pool of 14 blocks per node (two conversations' worth) serves 6
    conversations, every request completes, the coverage invariant holds at
    every turn completion and the pools are empty after the trace."""
    job = dev_job("1P_1D", x, n=6)
    for i, c in enumerate(job["conversations"]):  # all six in flight together
        c["arrival"] = 1e-4 * i
    job["device"]["kv_blocks_per_node"] = 14
    r = E.run(job)
    recs = E.records(r)
    assert len(recs) == 18 and all(v["status"] == "completed" for v in recs)
    life = r["device"]["kv_lifecycle"]
    assert life["blocks_in_use_at_end"] == 0 and life["coverage_errors"] == 0
    assert life["released_tables"] >= 6
    assert all(n["kv_blocks_peak"] <= 14 for n in r["device"]["nodes"])
    assert sum(n["admission_waits"] + n["stalled_rows"] for n in r["device"]["nodes"]) > 0


def test_flush_and_hop_race_keeps_coverage(gpu):
    """a turn's completion flush (KV-only row of its last token) may
    still be in flight on D when the next turn's P-path hop lands. Mixed
    routing with short P-path turns next to long D-local appends on the same D:
    the covered-token count must stay exact (no hole, no overrun)."""
    convs = [{"conv_id": "long", "arrival": 0.0, "turns": [[600, 3], [900, 3], [900, 3]]}]
    convs += [{"conv_id": f"s{i}", "arrival": 0.0005 * i, "turns": [[20, 2]] * 5} for i in range(6)]
    for x in (0.0, 0.5):
        job = {"cluster": "1P_1D", "x": x, "clock": "device", "conversations": convs,
               "device": {"model": "tiny", "weight_seed": 5, "token_seed": 9, "gpus": [0],
                          "prefill_chunk": 1024}}
        r = E.run(job)
        assert all(v["status"] == "completed" for v in E.records(r))
        assert r["device"]["kv_lifecycle"]["coverage_errors"] == 0


def test_shared_weights_per_gpu(gpu):
    """Nodes colocated on one GPU with the same model share one weight copy."""
    r = E.run(dev_job("2P_6D", 1.0, n=2))
    assert all(n["weights_shared_by"] == 8 for n in r["device"]["nodes"])


@pytest.mark.parametrize("cluster,x", [("1P_1D", 0.0), ("1P_1D", 1.0), ("4P_4D", 0.0), ("2P_6D", 0.5)])
def test_realtime_engine_tokens_match_oracle(gpu, cluster, x):
    """Wall-clock engine: a worker thread per node submits its steps, P->D hops
    are asynchronous copies retired by per-destination waiters. Every request
    completes with its target tokens and the generated ids equal the CPU
    oracle replaying the step log (copies applied where the engine issued them)."""
    r = E.run(rt_job(cluster, x, record_steps=True, n=4))
    recs = E.records(r)
    assert len(recs) == 12 and all(v["status"] == "completed" for v in recs)
    assert r["device"]["clock"] == "realtime"
    assert r["device"]["kv_lifecycle"]["coverage_errors"] == 0
    assert r["device"]["kv_lifecycle"]["blocks_in_use_at_end"] == 0
    if x < 1.0:
        assert r["link_transfers"] > 0 and r["device"]["kv_transfer"]["gbs"] > 0
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
            for p in range(e["start"], e["start"] + e["n"]):
                dst[e["dst_blocks"][p // 16], :, :, :, p % 16] = src[e["src_blocks"][p // 16], :, :, :, p % 16]
            continue
        pool = pools.setdefault(e["node"], O.KvPool(cfg, nblocks))
        n = len(e["q_len"])
        bt = np.array(e["block_tables"], dtype=np.int32).reshape(n, e["max_blocks"])
        t_o, _, margin = model.step(pool, e["q_len"], e["ctx"], e["tokens"], bt, want_logits=False)
        for i in range(n):
            if e["want"][i] and margin[i] > MARGIN:
                assert e["out"][i] == t_o[i], (e["node"], i, e["out"][i], t_o[i], margin[i])
                checked += 1
    assert checked > 20


def test_phase1_table_on_device_then_dynamic_routing(gpu):
    """§8f-1: Phase 1 of Algorithm 1 built with engine::device_benchmark_runner
    (every (key, x) cell runs on the GPU through the device clock), then the
    dynamic router consumes that table on the device clock."""
    import json as _json
    dev = {"model": "tiny", "weight_seed": 5, "token_seed": 9, "gpus": [0], "prefill_chunk": 512}
    keys = ["small|balanced|0.5", "small|balanced|1"]
    t = E.run({"op": "build_table", "clock": "device", "cluster": "1P_1D", "duration_s": 1.0, "grid_keys": keys,
               "device": dev})
    entries = _json.loads(t["table_json"])["entries"]
    assert sorted(entries) == sorted(keys)
    assert all(e["available"] and e["ttft_x0"] > 0 and e["tpot_x1"] > 0 for e in entries.values())
    wl = {"id": "w", "turn1": [256, 8], "turn2plus": [256, 8], "num_turns": 3, "qps": 1.0, "duration_s": 2.0}
    r = E.run({"cluster": "1P_1D", "policy": "dynamic", "table_json": t["table_json"], "clock": "device",
               "workload": wl, "seed": 1, "device": dev})
    recs = E.records(r)
    assert recs and all(v["status"] == "completed" for v in recs)
    assert sum(r["route_decisions"]) == sum(1 for v in recs if v["route"] == "D_local")


def test_next_turn_joins_the_next_iteration(gpu):
    """Iteration boundary (engine.cpp iter_done -> Ev::kick): a conversation's
    next turn, issued at the instant its predecessor completes (think time 0),
    rides in the very next step of its decode node instead of waiting one
    step behind it: every D-local append's final chunk starts at its arrival
    whenever the node was not already busy with another prefill chunk."""
    wl = {"id": "kick", "turn1": [48, 12], "turn2plus": [40, 12], "num_turns": 3, "qps": 4.0, "duration_s": 2.0}
    job = {"cluster": "1P_1D", "x": 1.0, "clock": "device", "seed": 5, "workload": wl,
           "device": {"model": "tiny", "weight_seed": 3, "token_seed": 4, "gpus": [0, 0], "kv_blocks_per_node": 0,
                      "prefill_chunk": 64, "record_tokens": False, "record_steps": True}}
    r = E.run(job)
    steps = [st for st in r["device"]["step_log"] if not st.get("copy")]
    appends = [st for st in steps if st.get("chunk_req") and st["chunk_req"]["turn"] >= 2 and st["chunk_req"]["final"]]
    assert len(appends) >= 5
    waits = [st["t_start"] - st["chunk_req"]["arrival"] for st in appends]
    assert sum(w < 1e-9 for w in waits) >= 0.8 * len(waits), waits
