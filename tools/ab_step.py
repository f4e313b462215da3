"""In-process A/B of the headline decode step (Llama-3-8B shape, B=200 at ctx
1024, random KV) across tuning configurations and/or builds of
libppd_b200.so: configurations alternate round by round so clock / power
drift hits all of them alike; reports the median device ms per step of each.

  PPD_AB="base:;nofuse:mlp_fused=0;old:@old_build/<sha>/paper_2603_13358_b200/libppd_b200.so" \
      python tools/ab_step.py
Each item is name:knob=v,...[@lib path]. One device (weights + KV pool) per build.
PPD_AB_MIX="m:n[,m:n...]" adds prefill rows (m new tokens over n cached) to
every step: the mixed decode + append / full prefill step of the
interference sweep.
"""
import contextlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2603_13358_b200 as ppd  # noqa: E402

DEFAULTS = {"gemm_pair": -1, "gemm_sched": -1, "gemm_stages": 0, "mlp_fused": 2, "attn_fused": 1,
            "gemm_occ2": 0, "gemm_multi_sub": 1, "attn_pf_ctas": 0, "pdl_overlap": 0, "gemm_l2_pre": 0,
            "layer_kernel": 0, "layer_l2_ahead": 16, "layer_stages": 0, "gemm_epi_pipe": 1, "l2_hint": 3}


def parse(spec):
    cfgs = []
    for item in spec.split(";"):
        if not item.strip():
            continue
        name, _, rest = item.partition(":")
        kv, _, path = rest.partition("@")
        knobs = {}
        for pair in filter(None, kv.split(",")):
            k, v = pair.split("=")
            knobs[k.strip()] = int(v)
        cfgs.append((name.strip(), knobs, path.strip() or ppd.LIB_PATH))
    return cfgs


@contextlib.contextmanager
def using(L):
    saved = ppd._lib
    ppd._lib = L
    try:
        yield
    finally:
        ppd._lib = saved


def main():
    import torch
    cfgs = parse(os.environ.get("PPD_AB", "base:;nofuse:mlp_fused=0"))
    rounds = int(os.environ.get("PPD_AB_ROUNDS", "8"))
    steps = int(os.environ.get("PPD_AB_STEPS", "4"))
    B, ctx0, BT = int(os.environ.get("PPD_AB_B", "200")), int(os.environ.get("PPD_AB_CTX", "1024")), 16
    cfg = ppd.qwen32b_cfg() if os.environ.get("PPD_AB_MODEL") == "qwen32b" else ppd.llama8b_cfg()
    max_ctx = ctx0 + rounds * len(cfgs) * (steps + 2) + 16
    bps = (max_ctx + BT - 1) // BT
    mix = [tuple(int(x) for x in it.split(":")) for it in filter(None, os.environ.get("PPD_AB_MIX", "").split(","))]
    mbps = max([bps] + [(m + n + BT - 1) // BT for m, n in mix])
    bts = np.zeros((B + len(mix), mbps), dtype=np.int32)
    bts[:B, :bps] = np.arange(B * bps, dtype=np.int32).reshape(B, bps)
    nxt = B * bps
    for j, (m, n) in enumerate(mix):
        k = (m + n + BT - 1) // BT
        bts[B + j, :k] = np.arange(nxt, nxt + k)
        nxt += k
    rng = np.random.default_rng(0)
    libs, devs = {}, {}
    for _, _, path in cfgs:
        if path in libs:
            continue
        libs[path] = ppd.load_lib(path, strict=False)
        with using(libs[path]):
            dev = ppd.Device(0, cfg, max_step_tokens=4096, max_step_seqs=256)
            dev.load_random_weights(1234)
            dev.kv_pool_init(nxt)
            ptr, nbytes = dev.kv_pool_ptr()
            ppd.check(libs[path].ppd_op_fill_random(ptr, nbytes // 2, 1234, 99, 0, None))
        devs[path] = dev
    tok = rng.integers(0, cfg.vocab, B).astype(np.int32)
    ctx = np.full(B, ctx0, dtype=np.int32)
    res = {name: [] for name, _, _ in cfgs}
    for _ in range(rounds):
        for name, knobs, path in cfgs:
            L = libs[path]
            with using(L):
                if hasattr(L, "ppd_set_tuning"):
                    for k, v in {**DEFAULTS, **knobs}.items():
                        if L.ppd_set_tuning(k.encode(), v) != 0 and k in knobs:
                            raise SystemExit(f"{name}: knob {k} rejected: {L.ppd_last_error().decode()}")
                for i in range(steps + 2):  # 2 warm-up steps: graph capture
                    q = [1] * B + [m for m, _ in mix]
                    c = list(ctx) + [n for _, n in mix]
                    toks = np.concatenate([tok] + [rng.integers(0, cfg.vocab, m) for m, _ in mix]).astype(np.int32)
                    r = devs[path].step(q, c, toks, bts, [1] * B + [0] * len(mix))
                    tok = r.tokens[:B]
                    ctx += 1
                    if i >= 2:
                        res[name].append(r.ms)
    torch.cuda.synchronize()
    out = {name: {"median_ms": float(np.median(v)), "min_ms": float(np.min(v)), "n": len(v)}
           for name, v in res.items()}
    base = out[cfgs[0][0]]["median_ms"]
    for name in out:
        out[name]["vs_first"] = out[name]["median_ms"] / base
    print(json.dumps(out))
    for path, dev in devs.items():
        with using(libs[path]):
            dev.close()


if __name__ == "__main__":
    main()
