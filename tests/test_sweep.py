"""§8f-2 / §8f-4 widening: the experiment grid (sweep harness) and the
analyses the paper's tables come from, plus real-trace ingest — each checked
against the UNMODIFIED reference (oracle/_ref/ref_tool) on the same jobs:

  * SweepPlan::full_default serialisation + hash (manifest compatibility)
  * run_sweep cells, results CSV, seed means, winner distribution (rendered
    table byte for byte) and compare_modes rows on a small plan
  * the resumable manifest: cells written by either tool are read by the other
  * failed cells (bad shape) recorded, sweep continues
  * pareto_frontier and winner_distribution on random inputs (ties, duplicates,
    degraded cells, error conditions)
  * weight_sweep (Phase-1 tables per SLO weight, dynamic replays)
  * ingest_trace filters / deterministic sampling / error text
All on the virtual clock (CPU); the device-clock sweep is in test_gpu_engine.py."""
import json
import math
import os
import random

import pytest

from oracle import oracle as O
from paper_2603_13358_b200 import engine as E


def default_plan():
    return json.loads(E.run({"op": "plan_default"})["plan_json"])


def small_plan(configs=None, duration=4.0):
    full = default_plan()
    wl = [w for w in full["workloads"] if w["id"] in ("dh1_short", "ph1_short")]
    return {"schema_version": 1,
            "configs": configs or [{"shape": "4R", "x_mode": "replica"}, {"shape": "1P_3D", "x_mode": "x0"},
                                   {"shape": "1P_3D", "x_mode": "x1"}, {"shape": "2P_2D", "x_mode": "x1/2"},
                                   {"shape": "1R_1P_2D", "x_mode": "x1"}],
            "workloads": wl, "qps_levels": [1.0, 4.0, 12.0], "seeds": [1, 2], "duration_s": duration}


def test_default_plan_matches_reference():
    ours, ref = E.run({"op": "plan_default"}), O.ref_tool({"op": "plan_default"})
    assert ours["plan_json"] == ref["plan_json"]
    assert ours["hash"] == ref["hash"]
    assert ours["cell_count"] == ref["cell_count"] == 17 * 18 * 10 * 3


def test_sweep_matches_reference():
    job = {"op": "sweep", "plan": small_plan(), "parallelism": 4,
           "compare": [["x0", "x1", "ttft_t2_mean"], ["x0", "x1", "tpot_mean"], ["x0", "x1", "tps"]]}
    ours, ref = E.run(job), O.ref_tool(job)
    for k in ("plan_hash", "calibration_hash", "cells", "csv", "means", "winner", "compare"):
        assert ours[k] == ref[k], k
    assert len(ours["cells"]) == 5 * 2 * 3 * 2
    assert not any(c["failed"] for c in ours["cells"])
    assert ours["winner"]["render"].startswith("Mode        TTFT")


def test_manifest_is_shared_with_reference(tmp_path):
    job = {"op": "sweep", "plan": small_plan(duration=3.0), "parallelism": 2}
    ref_dir, our_dir = tmp_path / "ref", tmp_path / "ours"
    ref = O.ref_tool({**job, "manifest_dir": str(ref_dir)})
    files = sorted(os.listdir(ref_dir))
    assert len(files) == len(ref["cells"])
    # ours resumes entirely from the reference's manifest ...
    assert E.run({**job, "manifest_dir": str(ref_dir)})["cells"] == ref["cells"]
    # ... and a partial manifest of ours is completed to the same cells
    ours = E.run({**job, "manifest_dir": str(our_dir)})
    assert sorted(os.listdir(our_dir)) == files
    for f in files[::2]:
        os.remove(our_dir / f)
    again = E.run({**job, "manifest_dir": str(our_dir)})
    assert again["cells"] == ours["cells"] == ref["cells"]
    for f in files:  # byte-identical cell files
        assert (our_dir / f).read_text() == (ref_dir / f).read_text()


def test_failed_cells_are_recorded():
    plan = small_plan(configs=[{"shape": "1P_3D", "x_mode": "x0"}, {"shape": "9Q", "x_mode": "x1"}])
    job = {"op": "sweep", "plan": plan}
    ours, ref = E.run(job), O.ref_tool(job)
    assert ours["cells"] == ref["cells"]
    bad = [c for c in ours["cells"] if c["failed"]]
    assert len(bad) == 12 and all(c["error"] for c in bad)
    assert ours["csv"] == ref["csv"]


@pytest.mark.parametrize("par", [1, 3])
def test_bad_x_mode_rejected_like_reference(par):
    """An unparsable x_mode aborts the sweep (the reference classifies a cell
    outside its per-cell try); ours also surfaces it from worker threads."""
    plan = small_plan(configs=[{"shape": "1P_3D", "x_mode": "x0"}, {"shape": "1P_3D", "x_mode": "y1"}])
    with pytest.raises(ValueError, match="bad x_mode: y1"):
        E.run({"op": "sweep", "plan": plan, "parallelism": par})
    if par == 1:  # the reference std::terminate()s when this happens on a worker thread
        with pytest.raises(RuntimeError, match="bad x_mode: y1"):
            O.ref_tool({"op": "sweep", "plan": plan})


def rand_points(rng, n):
    pts = []
    for i in range(n):
        if pts and rng.random() < 0.2:
            t, s, _ = rng.choice(pts)  # duplicate coordinates
        else:
            t, s = round(rng.uniform(0.1, 2.0), 1), float(rng.randint(1, 8) * 100)
        pts.append([t, s, f"c{i}"])
    return pts


def test_pareto_matches_reference():
    rng = random.Random(3)
    for n in (1, 2, 5, 17, 60):
        for _ in range(20):
            job = {"op": "pareto", "points": rand_points(rng, n)}
            assert E.run(job) == O.ref_tool(job)
    with pytest.raises(ValueError):
        E.run({"op": "pareto", "points": []})
    with pytest.raises(RuntimeError):
        O.ref_tool({"op": "pareto", "points": []})


def rand_cells(rng, n_cells, n_cfg):
    cats = ["Replica", "x=0", "0<x<1", "x=1", "hybrid"]
    out = []
    for c in range(n_cells):
        for k in range(n_cfg):
            m = {"tps": float(rng.choice([100, 200, 300])), "success_rate": rng.choice([1.0, 0.97, 0.5]),
                 "total_requests": 10, "completed_requests": 9}
            m["degraded"] = m["success_rate"] < 0.95
            if rng.random() < 0.9:
                m["ttft_t2_mean"] = rng.choice([0.1, 0.2, 0.3])
            if rng.random() < 0.9:
                m["tpot_mean"] = rng.choice([0.01, 0.02])
            out.append({"workload_id": f"w{c % 3}", "qps": float(c // 3 + 1), "config_label": f"cfg{k}",
                        "category": rng.choice(cats), "metrics": m})
    return out


def test_winner_distribution_matches_reference():
    rng = random.Random(5)
    for _ in range(30):
        job = {"op": "winner", "cells": rand_cells(rng, rng.randint(1, 9), rng.randint(2, 5))}
        assert E.run(job) == O.ref_tool(job)
    lonely = {"op": "winner", "cells": rand_cells(rng, 1, 1)}
    with pytest.raises(ValueError):
        E.run(lonely)
    with pytest.raises(RuntimeError):
        O.ref_tool(lonely)


def test_weight_sweep_matches_reference():
    base = next(w for w in default_plan()["workloads"] if w["id"] == "bal1_short")
    base = {**base, "duration_s": 4.0}
    job = {"op": "weight_sweep", "shape": "1P_3D", "base": base, "qps_levels": [1.0, 4.0],
           "w_tpot_list": [0.5, 1.0, 4.0], "seeds": [1],
           "grid_keys": ["small|balanced|1", "small|balanced|4", "medium|balanced|1", "medium|balanced|4"]}
    ours, ref = E.run(job), O.ref_tool(job)
    assert ours == ref
    assert len(ours["rows"]) == 3


def trace_jsonl(rng, n):
    lines = []
    for i in range(n):
        turns = [{"input_tokens": rng.randint(1, 3000), "output_tokens": rng.randint(1, 600)}
                 for _ in range(rng.randint(1, 6))]
        lines.append(json.dumps({"conv_id": f"conv-{i}", "turns": turns}))
        if rng.random() < 0.1:
            lines.append("")
    return "\n".join(lines) + "\n"


@pytest.mark.parametrize("filt", [{}, {"min_turns": 3}, {"min_ratio": 2.0}, {"sample_size": 7, "sample_seed": 9},
                                  {"min_turns": 1, "sample_size": 500, "sample_seed": 1}])
def test_ingest_trace_matches_reference(filt):
    text = trace_jsonl(random.Random(11), 60)
    job = {"op": "ingest_trace", "trace_jsonl": text, **filt}
    ours, ref = E.run(job), O.ref_tool(job)
    assert ours == ref
    assert ours["conversations"] or filt.get("min_ratio")


@pytest.mark.parametrize("bad", ['{"conv_id": "a"}', "not json", '{"conv_id": "a", "turns": [{"input_tokens": 0, '
                                                                  '"output_tokens": 1}]}'])
def test_ingest_trace_errors_match_reference(bad):
    job = {"op": "ingest_trace", "trace_jsonl": bad + "\n"}
    with pytest.raises(RuntimeError) as r:
        O.ref_tool(job)
    with pytest.raises((ValueError, RuntimeError)) as o:
        E.run(job)
    assert str(o.value) == str(r.value)


def test_compare_modes_nan_bands():
    # a plan whose QPS levels miss the high band: NaN (null) there in both tools
    plan = {**small_plan(), "qps_levels": [1.0, 4.0]}
    job = {"op": "sweep", "plan": plan, "compare": [["x0", "x1", "ttft_t2_mean"]]}
    ours = E.run(job)
    rows = ours["compare"]["x0|x1|ttft_t2_mean"]
    assert rows and rows[0][3] is None and rows[0][6] == 0
    assert ours["compare"] == O.ref_tool(job)["compare"]
    assert not any(isinstance(v, float) and math.isnan(v) for v in rows[0][1:3])


@pytest.mark.parametrize("cluster,x,qps", [("1P_3D", 0.0, 2.0), ("2P_2D", 1.0, 6.0), ("1R_1P_2D", 0.5, 4.0)])
def test_trace_replay_matches_reference(cluster, x, qps):
    """§8f-4: a ShareGPT-shaped JSONL trace, ingested (filters + sampling) and
    replayed at a target QPS, gives the reference's records byte for byte."""
    text = trace_jsonl(random.Random(21), 80)
    job = {"cluster": cluster, "x": x, "trace_jsonl": text, "min_turns": 2, "sample_size": 30, "sample_seed": 4,
           "qps_replay": qps, "seed": 7}
    ours, ref = E.run({"op": "simulate", **job}), O.ref_tool({"op": "simulate", **job})
    assert ours["records_jsonl"] == ref["records_jsonl"]
    for k in ("link_transfers", "link_bytes", "makespan", "node_stats"):
        assert ours[k] == ref[k], k
    assert len(E.records(ours)) > 30
