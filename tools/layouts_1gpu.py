"""configs[3]-shape run of the 8-node layouts (2P_6D, 4P_4D) with every node on
ONE B200 (functional + device-clock evidence when only one GPU is available):
PD (x=0) vs PPD (x=1) turn-2+ TTFT / TPOT and the P->D link statistics, Llama-3-8B
shape, 3 turns of (2048, 128) then 2 x (1024, 128). Each node's clock advances
by its own CUDA-event time; nodes sharing the GPU serialise on it, so this is
not a multi-GPU throughput number. PPD_LAYOUT_QPS / PPD_LAYOUT_DUR override
the load (default 8 qps for 4 s)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_13358_b200 import engine as E  # noqa: E402


def main():
    import paper_2603_13358_b200 as ppd
    os.environ.setdefault("PPD_DUMP_BAD_STEP", "gpurun_out/bad_step.json")
    for kv in filter(None, os.environ.get("PPD_LAYOUT_KNOBS", "").split(",")):
        k, v = kv.split("=")
        ppd.check(ppd.lib().ppd_set_tuning(k.encode(), int(v)))
    qps = float(os.environ.get("PPD_LAYOUT_QPS", "8"))
    dur = float(os.environ.get("PPD_LAYOUT_DUR", "4"))
    wl = {"id": "cfg4", "turn1": [2048, 128], "turn2plus": [1024, 128], "num_turns": 3, "qps": qps,
          "duration_s": dur}
    for layout in os.environ.get("PPD_LAYOUTS", "2P_6D,4P_4D").split(","):
        out = {"cluster": layout, "workload": wl, "gpus": "all nodes on GPU 0"}
        for x in (0.0, 1.0):
            job = {"cluster": layout, "x": x, "clock": "device", "seed": 3, "workload": wl,
                   "device": {"model": "llama8b", "weight_seed": 20260313, "token_seed": 3, "gpus": [0],
                              "kv_blocks_per_node": int(os.environ.get("PPD_LAYOUT_KV", "2000")), "prefill_chunk": 2048,
                              "record_tokens": False}}
            t0 = time.perf_counter()
            try:
                r = E.run(job)
            except Exception as e:  # report and continue with the next run
                print(json.dumps({"cluster": layout, "x": x, "error": str(e)}), flush=True)
                continue
            a = r["aggregate"]
            ms = lambda v: None if v is None else round(v * 1e3, 2)
            out[f"x{int(x)}"] = {"ttft_t2_p50_ms": ms(a["ttft_t2_p50"]), "ttft_t2_p99_ms": ms(a["ttft_t2_p99"]),
                                 "tpot_mean_ms": ms(a["tpot_mean"]), "success_rate": a["success_rate"],
                                 "link_transfers": r["link_transfers"], "link_gb": r["link_bytes"] / 1e9,
                                 "kv_transfer_gbs": r["device"]["kv_transfer"]["gbs"],
                                 "wall_s": round(time.perf_counter() - t0, 1)}
        if "x0" in out and "x1" in out:
            p50 = (out["x0"]["ttft_t2_p50_ms"], out["x1"]["ttft_t2_p50_ms"])
            out["ttft_t2_p50_reduction"] = None if None in p50 else 1 - p50[1] / p50[0]
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
