"""Timeline of one K8 decode layer kernel launch (layer 5 of the B=200,
ctx 1024 Llama-3-8B-shape decode step): per job, the spread over the 148 CTAs
of (activations ready at the producer, last MMA commit, epilogue arrival,
glue end), in microseconds from the earliest kernel entry. Uses the
layer_diag bit 256 probe (event times written into the KV pool's last 64 KB).

  PPD_K8_DIAG=256 python tools/k8_trace.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2603_13358_b200 as ppd  # noqa: E402


def main():
    diag = int(os.environ.get("PPD_K8_DIAG", "256"))
    B, ctx0, BT = int(os.environ.get("PPD_K8_B", "200")), 1024, 16
    cfg = ppd.llama8b_cfg()
    bps = (ctx0 + 64 + BT - 1) // BT
    dev = ppd.Device(0, cfg, max_step_tokens=4096, max_step_seqs=256)
    dev.load_random_weights(1234)
    nblk = B * bps + 2
    dev.kv_pool_init(nblk)
    ptr, nbytes = dev.kv_pool_ptr()
    ppd.check(ppd.lib().ppd_op_fill_random(ptr, nbytes // 2, 1234, 99, 0, None))
    bts = np.arange(B * bps, dtype=np.int32).reshape(B, bps)
    tok = np.random.default_rng(0).integers(0, cfg.vocab, B).astype(np.int32)
    ctx = np.full(B, ctx0, dtype=np.int32)
    ppd.check(ppd.lib().ppd_set_tuning(b"layer_diag", diag))
    out = {}
    for i in range(6):
        r = dev.step([1] * B, ctx, tok, bts)
        tok, ctx = r.tokens, ctx + 1
        out.setdefault("step_ms", []).append(r.ms)
    raw = dev.kv_pool_read(65536, nbytes - 65536).view(np.uint64)[: 148 * 20].reshape(148, 20).astype(np.float64)
    t0 = raw[:, 16].min()
    rel = (raw - t0) / 1000.0
    names = ["ready", "mma_done", "epi_arrive", "glue_end"]
    for j in range(4):
        for k, nm in enumerate(names):
            v = rel[:, 4 * j + k]
            out[f"job{j}_{nm}"] = [round(float(v.min()), 2), round(float(np.median(v)), 2), round(float(v.max()), 2)]
    out["entry_spread_us"] = round(float(rel[:, 16].max()), 2)
    out["pdl_wait_done"] = [round(float(rel[:, 0].min()), 2), round(float(rel[:, 0].max()), 2)]
    print(json.dumps(out))
    ppd.check(ppd.lib().ppd_set_tuning(b"layer_diag", 0))
    dev.close()


if __name__ == "__main__":
    main()
