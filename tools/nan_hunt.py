"""Repeat Llama-3-8B-shape steps of the shape that once produced a non-finite
logit in a device-clock layout run (1 decode row + a 1024-token append over
3328 cached, and variants) and check every sampled id / logit row is finite.
PPD_NH_KNOBS="k=v,..." sets tuning knobs first; PPD_NH_REPS repetitions."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_13358_b200 as ppd  # noqa: E402


def main():
    for kv in filter(None, os.environ.get("PPD_NH_KNOBS", "").split(",")):
        k, v = kv.split("=")
        ppd.check(ppd.lib().ppd_set_tuning(k.encode(), int(v)))
    reps = int(os.environ.get("PPD_NH_REPS", "40"))
    cfg = ppd.llama8b_cfg()
    dev = ppd.Device(0, cfg, max_step_tokens=2624, max_step_seqs=64)
    dev.load_random_weights(20260313)
    nblk = 4096
    dev.kv_pool_init(nblk)
    ptr, nbytes = dev.kv_pool_ptr()
    ppd.check(ppd.lib().ppd_op_fill_random(ptr, nbytes // 2, 3, 99, 0, None))
    rng = np.random.default_rng(0)
    cases = {"mix1+1024@3328": ([1, 1024], [3400, 3328]), "pf1024@3328": ([1024], [3328]),
             "mix8+1024@3328": ([1] * 8 + [1024], [3000 + 50 * i for i in range(8)] + [3328]),
             "mix1+1536@2048": ([1, 1536], [3400, 2048]), "pf2048@0": ([2048], [0])}
    bad = {}
    for name, (q, c) in cases.items():
        n = len(q)
        bt = np.zeros((n, 300), dtype=np.int32)
        for i in range(n):
            bt[i] = rng.permutation(nblk)[:300]
        nb = 0
        for r in range(reps):
            toks = rng.integers(0, cfg.vocab, int(sum(q))).astype(np.int32)
            res = dev.step(q, c, toks, bt)
            lg = dev.last_logits(n)
            ok = np.isfinite(lg).all() and all(0 <= t < cfg.vocab for t in res.tokens)
            nb += not ok
        bad[name] = nb
        print(json.dumps({"case": name, "reps": reps, "bad": nb}), flush=True)
    dev.close()


if __name__ == "__main__":
    main()
