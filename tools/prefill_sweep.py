"""Prefill-step profile on the GPU: one full prefill (or append) of the
Llama-3-8B shape through ppd_step with per-kernel-class CUDA-event timing.
Reports attention TFLOP/s (causal: 2 * n_q * n_keys_avg * Hq * Dh * 2 per layer)
and GEMM TFLOP/s. Run twice with PPD_ATTN_TC=1/0 to compare the tcgen05 and
mma.sync prefill attention."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_13358_b200 as ppd  # noqa: E402


def main():
    if os.environ.get("PPD_LIB"):  # A/B another build of libppd_b200.so
        ppd._lib = ppd.load_lib(os.environ["PPD_LIB"], strict=False)
    for kv in filter(None, os.environ.get("PPD_PF_KNOBS", "").split(",")):
        k, v = kv.split("=")
        ppd.check(ppd.lib().ppd_set_tuning(k.encode(), int(v)))
    cfg = ppd.llama8b_cfg()
    dev = ppd.Device(0, cfg, max_step_tokens=8192, max_step_seqs=8)
    dev.load_random_weights(1)
    dev.kv_pool_init(2048 + 64)
    ptr, nbytes = dev.kv_pool_ptr()
    ppd.check(ppd.lib().ppd_op_fill_random(ptr, nbytes // 2, 3, 99, 0, None))
    rng = np.random.default_rng(0)
    bt = np.arange(2048, dtype=np.int32)
    out = []
    cases = ((1024, 0), (4096, 0), (8192, 0), (1536, 6144), (2048, 14336), (2048, 30720))
    if os.environ.get("PPD_SWEEP"):
        m0, n0 = (int(v) for v in os.environ["PPD_SWEEP"].split(","))
        cases = ((m0, n0),)
    for m, n in cases:
        toks = rng.integers(0, cfg.vocab, m).astype(np.int32)
        dev.step([m], [n], toks, bt)  # warm
        dev.set_profiling(True)
        dev.reset_stats()
        for _ in range(3):
            dev.step([m], [n], toks, bt)
        st = dev.stats()
        dev.set_profiling(False)
        keys_avg = n + (m + 1) / 2
        attn_flop = 4.0 * m * keys_avg * cfg.n_q_heads * 128 * cfg.n_layers * 3
        lin = 2.0 * m * (4096 * 6144 + 4096 * 4096 + 4096 * 28672 + 14336 * 4096) * cfg.n_layers * 3
        res = {"m": m, "ctx": n, "step_ms": st["step_ms"] / 3, "attn_ms": st["attn_ms"] / 3,
               "gemm_ms": st["gemm_ms"] / 3,
               "attn_tflops": attn_flop / (st["attn_ms"] * 1e-3) / 1e12 if st["attn_ms"] else None,
               "gemm_tflops": lin / (st["gemm_ms"] * 1e-3) / 1e12 if st["gemm_ms"] else None,
               "tc_attention": os.environ.get("PPD_ATTN_TC", "1") != "0",
               "knobs": os.environ.get("PPD_PF_KNOBS", "")}
        out.append(res)
        print(json.dumps(res), flush=True)
    dev.close()


if __name__ == "__main__":
    main()
