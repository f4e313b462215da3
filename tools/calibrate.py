"""Device-measured calibration: time full prefill,
append prefill, decode steps and prefill-in-decode interference on the B200
through the C-ABI, fit the reference's CalibrationTable coefficients from them
(ppd::cost::fit_from_measurements), and build the Phase-1 decision table the
dynamic PPD router consumes from the fitted table.

  python tools/calibrate.py [--out profiles/calibration_r01.json]

Interference is measured the way the engine runs it: a full prefill of N
tokens rides in the decode step as ceil(N / chunk) chunks; an append of total
N tokens is m = 128 new tokens over N - 128 cached, in one step."""
import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import paper_2603_13358_b200 as ppd  # noqa: E402
from paper_2603_13358_b200 import engine as E  # noqa: E402

CHUNK = 2048


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(REPO, "profiles", "calibration_r01.json"))
    ap.add_argument("--gpu", type=int, default=0)
    args = ap.parse_args()
    cfg = ppd.llama8b_cfg()
    B, CTX = 200, 1024
    dev = ppd.Device(args.gpu, cfg, max_step_tokens=4 * CHUNK + 256 + 64, max_step_seqs=256)
    dev.load_random_weights(7)
    bps = (CTX + 64 + 15) // 16
    extra = 4 * 8192 // 16 + 64
    dev.kv_pool_init(B * bps + extra + 64)
    ptr, nbytes = dev.kv_pool_ptr()
    ppd.check(ppd.lib().ppd_op_fill_random(ptr, nbytes // 2, 3, 99, 0, None))
    rng = np.random.default_rng(0)
    bts = np.arange(B * bps, dtype=np.int32).reshape(B, bps)
    base = B * bps
    seq_blocks = [np.arange(base + i * 512, base + (i + 1) * 512, dtype=np.int32) for i in range(4)]

    def med(fn, n=3):
        fn()
        return float(np.median([fn() for _ in range(n)]))

    def step(q, c, bt, want=None):
        toks = rng.integers(0, cfg.vocab, int(np.sum(q))).astype(np.int32)
        return dev.step(q, c, toks, bt, want).ms

    samples = {"full": [], "append": [], "decode": [], "interference": []}
    t0 = time.time()
    for n in (256, 512, 1024, 2048, 4096, 8192):
        ms = 0.0
        for c0 in range(0, n, CHUNK):  # the engine's chunked full prefill
            m = min(CHUNK, n - c0)
            ms += med(lambda: step([m], [c0], seq_blocks[0]))
        samples["full"].append([n, ms * 1e-3])
    for m, n in ((128, 896), (256, 1792), (512, 3584), (1024, 3072), (1536, 6144), (128, 7936)):
        samples["append"].append([m, n, med(lambda: step([m], [n], seq_blocks[1])) * 1e-3])
    alone = {}
    for b in (1, 16, 64, 128, 200):
        alone[b] = med(lambda: step([1] * b, [CTX] * b, bts[:b]))
        samples["decode"].append([b, alone[b] * 1e-3])
    for b in (1, 200):
        for kind in ("full", "append"):
            for tokens in (1024, 8192):
                for conc in (1, 4):
                    bt = np.zeros((b + conc, max(bps, 512)), dtype=np.int32)
                    bt[:b, :bps] = bts[:b]
                    for i in range(conc):
                        bt[b + i, :512] = seq_blocks[i]
                    if kind == "full":
                        chunks = [(c0, min(CHUNK, tokens - c0)) for c0 in range(0, tokens, CHUNK)]
                        ms = np.mean([med(lambda: step([1] * b + [m] * conc, [CTX] * b + [c0] * conc, bt,
                                                       [1] * b + [0] * conc)) for c0, m in chunks])
                    else:
                        ms = med(lambda: step([1] * b + [128] * conc, [CTX] * b + [tokens - 128] * conc, bt,
                                              [1] * b + [0] * conc))
                    samples["interference"].append({"kind": kind, "prefill_tokens": tokens, "concurrent_prefills": conc,
                                                    "decode_batch": b, "tpot_multiplier": float(ms / alone[b])})
    kvb = ppd.kv_block_bytes(cfg) / 16
    samples["kv_bytes_per_token"] = kvb
    measure_s = time.time() - t0
    dev.close()
    fit = E.run({"op": "fit_calibration", "samples": samples})
    table = E.run({"op": "build_table", "calib_json": fit["calib_json"], "cluster": "1P_3D", "seeds": [1, 2],
                   "duration_s": 10.0})
    tj = json.loads(table["table_json"])
    out = {"model": "llama-3-8b-shape", "gpu": "B200", "chunk_tokens": CHUNK, "samples": samples,
           "calibration": json.loads(fit["calib_json"]), "calibration_hash": fit["hash"],
           "decision_table": tj, "x_star_1_keys": sum(e["x_star"] for e in tj["entries"].values()),
           "measure_s": measure_s}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(out, open(args.out, "w"), indent=1)
    c = out["calibration"]
    print(json.dumps({"full_a_lin": c["full_a_lin"], "full_b_quad": c["full_b_quad"], "append_a_lin": c["append_a_lin"],
                      "append_b_cross": c["append_b_cross"], "decode_c_base": c["decode_c_base"],
                      "decode_d_batch": c["decode_d_batch"], "x_star_1_keys": out["x_star_1_keys"],
                      "interference": [(p["kind"], p["prefill_tokens"], p["concurrent_prefills"], p["decode_batch"],
                                        round(p["tpot_multiplier"], 3)) for p in samples["interference"]]}))


if __name__ == "__main__":
    main()
