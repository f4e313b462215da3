"""Device-engine stress with the tiny model: every (layout, routing x, prefill
chunk, load) combination on GPU 0 must complete every request."""
import sys, json, itertools
sys.path.insert(0, '.')
from paper_2603_13358_b200 import engine as E
bad = 0
for cluster, x, chunk, qps in itertools.product(["2P_6D", "4P_4D", "1P_3D"], [0.0, 1.0], [16, 64], [40.0, 120.0]):
    wl = {"id": "s", "turn1": [96, 6], "turn2plus": [48, 6], "num_turns": 3, "qps": qps, "duration_s": 1.0}
    job = {"cluster": cluster, "x": x, "clock": "device", "seed": 3, "workload": wl,
           "device": {"model": "tiny", "weight_seed": 5, "token_seed": 9, "gpus": [0], "prefill_chunk": chunk}}
    try:
        r = E.run(job)
        recs = E.records(r)
        ok = all(v["status"] == "completed" for v in recs)
        print(cluster, x, chunk, qps, len(recs), ok, flush=True)
        bad += not ok
    except Exception as e:
        print(cluster, x, chunk, qps, "ERROR", e, flush=True)
        bad += 1
print("bad", bad)
