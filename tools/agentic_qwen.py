"""BASELINE configs[4] on the device clock: Qwen2.5-32B shape (GQA 40/8, QKV
bias, random-init bf16), a long multi-turn agentic trace (8 turns: 4096 in,
then 7 x 1536 in, context growing past 16k tokens), 2P_6D, fixed-fraction
routing x in {0, 1/3, 1/2, 2/3, 1} vs dynamic PPD whose Phase-1 table
(routing.cpp:220-244) is built from DEVICE runs (engine::device_benchmark_runner
through op=build_table clock=device) -- the reference's sweep.cpp:456-547
experiment with every prefill, decode iteration and KV hop executed on a B200.

One GPU here: all 8 nodes share it (one copy of the 65.5 GB of weights per
GPU, per-node KV pools); each node's clock advances by its own CUDA-event
time. Output tokens per turn are 64 (configs[4] does not fix them; 512 would
make each 1-GPU run ~8x longer without changing the context growth, which
comes from the input tokens). Prints one JSON object.
  python tools/agentic_qwen.py [--quick] [--out profiles/agentic_qwen_r02.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_13358_b200 import engine as E  # noqa: E402


def summary(r, t0):
    a = r["aggregate"]
    recs = E.records(r)
    t2 = [x for x in recs if x["turn_index"] >= 2]
    ms = lambda v: None if v is None else v * 1e3
    return {"ttft_t2_p50_ms": ms(a["ttft_t2_p50"]), "ttft_t2_p99_ms": ms(a["ttft_t2_p99"]),
            "ttft_t2_mean_ms": ms(a["ttft_t2_mean"]), "tpot_mean_ms": ms(a["tpot_mean"]),
            "success_rate": a["success_rate"], "turns": len(recs), "turn2plus": len(t2),
            "d_local_ratio": (sum(1 for x in t2 if x["route"] == "D_local") / len(t2)) if t2 else None,
            "link_transfers": r["link_transfers"], "link_gb": r["link_bytes"] / 1e9,
            "kv_transfer_gbs": r["device"]["kv_transfer"]["gbs"], "wall_s": time.perf_counter() - t0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--out", default="")
    ap.add_argument("--qps", type=float, default=0.5)
    ap.add_argument("--duration", type=float, default=8.0)
    ap.add_argument("--seed", type=int, default=1)
    args = ap.parse_args()
    out_tok = 16 if args.quick else 64
    wl = {"id": "cfg5_agentic", "turn1": [4096, out_tok], "turn2plus": [1536, out_tok],
          "num_turns": 4 if args.quick else 8, "qps": args.qps,
          "duration_s": 4.0 if args.quick else args.duration}
    # 8 nodes on one GPU: 65.5 GB of shared weights + 8 KV pools of 2600 x 4 MiB blocks
    dev = {"model": "qwen32b", "weight_seed": 1234, "token_seed": 5, "gpus": [0], "prefill_chunk": 2048,
           "p_prefill_chunk": 8192, "kv_blocks_per_node": 2600, "record_tokens": False}
    res = {"config": "BASELINE configs[4] (Qwen2.5-32B shape, 2P_6D, agentic multi-turn)", "workload": wl,
           "device": dev, "clock": "device", "placement": "all 8 nodes on GPU 0 (1 GPU per gpurun call)"}
    # Phase 1 on the device: the keys this trace reaches (turn 2+ are prefill-heavy;
    # context medium (4k-16k) then large (>= 16k); qps bin of the trace)
    t0 = time.perf_counter()
    qbin = 0.5 if args.qps < 0.75 else 1.0
    keys = [f"medium|prefill_heavy|{qbin:g}", f"large|prefill_heavy|{qbin:g}"]
    tab = E.run({"op": "build_table", "clock": "device", "cluster": "2P_6D", "grid_keys": keys,
                 "duration_s": 3.0 if args.quick else 6.0, "device": dev})
    res["phase1"] = {"keys": keys, "entries": json.loads(tab["table_json"])["entries"],
                     "wall_s": time.perf_counter() - t0}
    runs = {}
    for name, extra in [("x0", {"x": 0.0}), ("x1/3", {"x": 1 / 3}), ("x1/2", {"x": 0.5}), ("x2/3", {"x": 2 / 3}),
                        ("x1", {"x": 1.0}), ("dynamic", {"policy": "dynamic", "table_json": tab["table_json"]})]:
        t0 = time.perf_counter()
        r = E.run({"cluster": "2P_6D", "clock": "device", "workload": wl, "seed": args.seed, "device": dev, **extra})
        runs[name] = summary(r, t0)
        print(name, json.dumps(runs[name]), file=sys.stderr, flush=True)
    res["runs"] = runs
    base = runs["x0"]["ttft_t2_p50_ms"]
    res["ttft_t2_p50_reduction_vs_x0"] = {k: (1 - v["ttft_t2_p50_ms"] / base) if base and v["ttft_t2_p50_ms"] else None
                                          for k, v in runs.items()}
    s = json.dumps(res)
    print(s)
    if args.out:
        with open(args.out, "w") as f:
            f.write(s + "\n")


if __name__ == "__main__":
    main()
