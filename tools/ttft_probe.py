"""Where does turn-2+ TTFT go? Runs bench.py's 1P_1D device-clock trace for
x=0 (PD) and x=1 (PPD) with the step log on and prints, per turn-2+
request, its TTFT, plus the distribution of step durations by kind
(decode-only / with a prefill chunk) and the chunk sizes."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_13358_b200 import engine as E  # noqa: E402


def main():
    wl = {"id": "cfg3", "turn1": [1536, 512], "turn2plus": [1536, 512], "num_turns": 4, "qps": 1.0,
          "duration_s": float(os.environ.get("PPD_TP_DUR", "12"))}
    for x in (0.0, 1.0):
        job = {"cluster": "1P_1D", "x": x, "clock": "device", "seed": 3, "workload": wl,
               "device": {"model": "llama8b", "weight_seed": 20260313, "token_seed": 3, "gpus": [0, 0],
                          "kv_blocks_per_node": 8192, "prefill_chunk": int(os.environ.get("PPD_TP_CHUNK", "2048")),
                          "record_tokens": False, "record_steps": True}}
        r = E.run(job)
        recs = E.records(r)
        t2 = sorted([(rc["arrival"], rc["turn_index"], (rc["first_token"] - rc["arrival"]) * 1e3)
                     for rc in recs if rc["turn_index"] >= 2 and rc.get("first_token") is not None])
        steps = [s for s in r.get("device", {}).get("step_log", []) if not s.get("copy")]
        big = [(s["node"], sum(q for q in s["q_len"] if q > 1), len(s["q_len"]), round(s["ms"], 2)) for s in steps
               if max(s["q_len"]) > 1]
        dec = [s["ms"] for s in steps if max(s["q_len"]) == 1]
        # per final prefill chunk on a D node: queue wait (step start - arrival) and the step itself
        waits = [(s["chunk_req"]["turn"], round((s["t_start"] - s["chunk_req"]["arrival"]) * 1e3, 2), round(s["ms"], 2),
                  len(s["q_len"]) - 1)
                 for s in steps if s.get("chunk_req") and s["chunk_req"]["final"] and s["chunk_req"]["turn"] >= 2]
        print(json.dumps({"x": x, "turn2plus_final_chunks(turn,wait_ms,step_ms,decode_rows)": waits[:60]}))
        print(json.dumps({"x": x, "ttft_ms": [round(t[2], 1) for t in t2], "turns": [t[1] for t in t2],
                          "p50": float(np.median([t[2] for t in t2])),
                          "decode_step_ms_p50": float(np.median(dec)) if dec else None,
                          "prefill_steps(node,tokens,rows,ms)": big[:40],
                          "aggregate": {k: r["aggregate"][k] for k in ("ttft_t2_p50", "ttft_t2_p99", "tpot_mean")}}))


if __name__ == "__main__":
    main()
