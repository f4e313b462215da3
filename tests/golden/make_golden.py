"""Generates tests/golden/ref_records.json from the UNMODIFIED reference
(oracle/_ref/ref_tool, built from /root/reference/proj by oracle/Makefile).
Run here (the reference is not on the GPU box):  python tests/golden/make_golden.py
Each case stores the job and the reference's records JSONL, link accounting,
makespan, prefill waits and calibration hash; tests/test_engine_virtual.py
requires the engine's virtual clock to reproduce every field exactly."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402


def conv(cid, arrival, turns):
    return {"conv_id": cid, "arrival": arrival, "turns": [list(t) for t in turns]}


def cases():
    C = []
    # test_simulator.cpp known answers
    C.append(("replica_identity", {"cluster": "4R", "x": 0.0, "conversations": [conv("solo", 0.0, [(1000, 4)])]}))
    for x in (0.0, 1.0):
        C.append((f"pd_x{int(x)}", {"cluster": "1P_1D", "x": x,
                                    "conversations": [conv("c0", 0.0, [(1000, 4), (1000, 4)])]}))
        C.append((f"five_turn_x{int(x)}", {"cluster": "1P_1D", "x": x,
                                           "conversations": [conv("t", 0.0, [(512, 64)] * 5)]}))
    C.append(("conservation", {"cluster": "2P_2D", "x": 0.5, "seed": 5, "workload": {
        "id": "cons", "turn1": [512, 128], "turn2plus": [128, 128], "num_turns": 3, "qps": 4, "duration_s": 10}}))
    C.append(("determinism", {"cluster": "2P_2D", "x": 0.5, "seed": 9, "workload": {
        "id": "det", "turn1": [1024, 128], "turn2plus": [256, 256], "num_turns": 2, "qps": 6, "duration_s": 8}}))
    C.append(("timeout_slow_link", {"cluster": "1P_1D", "x": 0.0, "calib_overrides": {"link_bandwidth": 1e6},
                                    "conversations": [conv("late", 0.0, [(1000, 4)])]}))
    C.append(("think_time", {"cluster": "1P_1D", "x": 1.0, "think_time_s": 2.0,
                             "conversations": [conv("tt", 0.0, [(500, 4), (100, 4)])]}))
    C.append(("hybrid", {"cluster": "1R_1P_1D", "x": 1.0, "seed": 4, "workload": {
        "id": "hyb", "turn1": [512, 64], "turn2plus": [128, 64], "num_turns": 2, "qps": 6, "duration_s": 10}}))
    # acceptance.cpp fixtures
    for shape in ("1P_3D", "2P_2D", "3P_1D"):
        for x in (0.0, 1.0):
            C.append((f"throttled_{shape}_x{int(x)}", {"cluster": shape, "x": x, "seed": 11,
                                                        "calib_overrides": {"link_bandwidth": 1.4e9},
                                                        "workload": {"id": "saturate", "turn1": [1024, 64],
                                                                     "turn2plus": [1024, 64], "num_turns": 3,
                                                                     "qps": 12, "duration_s": 15}}))
    C.append(("mm1_exponential", {"cluster": "1R", "x": 0.0, "qps_replay": 0.5, "request_timeout_s": 1e9, "seed": 7,
                                  "calib_overrides": {"full_a_lin": 1.0, "full_b_quad": 0, "decode_c_base": 1e-9,
                                                      "decode_d_batch": 0,
                                                      "prefill_service_distribution": "exponential"},
                                  "conversations": [conv(f"q{i}", -1, [(1, 1)]) for i in range(800)]}))
    # BASELINE configs 3-5 shapes (virtual clock)
    for x in (0.0, 1.0 / 3, 0.5, 1.0):
        C.append((f"cfg5_2P_6D_x{x:.3f}", {"cluster": "2P_6D", "x": x, "seed": 2, "workload": {
            "id": "agentic", "turn1": [4096, 512], "turn2plus": [1536, 512], "num_turns": 8, "qps": 2,
            "duration_s": 10}}))
    for shape in ("2P_6D", "4P_4D"):
        for x in (0.0, 1.0):
            C.append((f"cfg4_{shape}_x{int(x)}", {"cluster": shape, "x": x, "seed": 1, "workload": {
                "id": "cfg4", "turn1": [2048, 128], "turn2plus": [1024, 128], "num_turns": 3, "qps": 16,
                "duration_s": 10}}))
    C.append(("cfg3_1P_1D_x1", {"cluster": "1P_1D", "x": 1.0, "seed": 3, "workload": {
        "id": "cfg3", "turn1": [1536, 512], "turn2plus": [1536, 512], "num_turns": 4, "qps": 1, "duration_s": 10}}))
    return C


def main():
    out = {"generator": "tests/golden/make_golden.py", "reference": "/root/reference/proj (unmodified)", "cases": []}
    for name, job in cases():
        job = dict(job, op="simulate")
        r = O.ref_tool(job)
        out["cases"].append({"name": name, "job": job, "records_jsonl": r["records_jsonl"],
                             "link_transfers": r["link_transfers"], "link_bytes": r["link_bytes"],
                             "link_queue_delays": r["link_queue_delays"], "makespan": r["makespan"],
                             "prefill_wait_samples": r["prefill_wait_samples"], "node_stats": r["node_stats"],
                             "session_miss_fallbacks": r["session_miss_fallbacks"], "calib_hash": r["calib_hash"]})
    path = os.path.join(HERE, "ref_records.json")
    with open(path, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print(path, len(out["cases"]), "cases", os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
