"""Turn-2+ TTFT p50, PD (x=0) vs PPD (x=1), over trace seeds {1, 2, 3} (the
reference sweep's default seeds, sweep.hpp:34): BASELINE configs[2] on 1P_1D,
Llama-3-8B shape, device clock, both nodes on GPU 0 -- the bench's TTFT
section with per-seed spread."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_13358_b200 import engine as E  # noqa: E402


def main():
    out = []
    for qps in (1.0, 2.0):
        wl = {"id": "cfg3", "turn1": [1536, 512], "turn2plus": [1536, 512], "num_turns": 4, "qps": qps,
              "duration_s": 12.0}
        for seed in (1, 2, 3):
            row = {"qps": qps, "seed": seed}
            for x in (0.0, 1.0):
                job = {"cluster": "1P_1D", "x": x, "clock": "device", "seed": seed, "workload": wl,
                       "device": {"model": "llama8b", "weight_seed": 20260313, "token_seed": 3, "gpus": [0, 0],
                                  "kv_blocks_per_node": 0, "prefill_chunk": 2048, "record_tokens": False}}
                a = E.run(job)["aggregate"]
                row[f"x{int(x)}_ttft_p50_ms"] = a["ttft_t2_p50"] * 1e3
                row[f"x{int(x)}_tpot_ms"] = a["tpot_mean"] * 1e3
            row["reduction"] = 1 - row["x1_ttft_p50_ms"] / row["x0_ttft_p50_ms"]
            out.append(row)
            print(json.dumps(row), flush=True)
    for qps in (1.0, 2.0):
        r = [o["reduction"] for o in out if o["qps"] == qps]
        print(json.dumps({"qps": qps, "mean_reduction": sum(r) / len(r), "min": min(r), "max": max(r)}), flush=True)


if __name__ == "__main__":
    main()
