"""Where the PPD turn-2+ TTFT goes: the D-node step that carries a 1536-token
append (configs[2]) next to a few decode rows, vs the P-node full prefills PD
runs instead (3584 / 5632 / 7680 tokens), on the Llama-3-8B shape. Per step:
device ms (CUDA events), the attention / GEMM split (profiling events) and the
achieved PFLOP/s; then the four projection GEMMs at the append's token count,
tcgen05 kernel vs cuBLAS. Prints JSON lines; PPD_PROFILE_ONLY=1 runs one
append step only (for an ncu launch list)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_13358_b200 as ppd  # noqa: E402

P_LIN = 6.98e9  # Llama-3-8B linear params (no embedding / lm_head)


def flops(q_len, ctx):
    f = 0.0
    for m, n in zip(q_len, ctx):
        f += 2 * P_LIN * m + 4 * 32 * 128 * 32 * (m * n + m * m / 2)
    return f


def main():
    cfg = ppd.llama8b_cfg()
    dev = ppd.Device(0, cfg, max_step_tokens=8448, max_step_seqs=64)
    dev.load_random_weights(7)
    dev.kv_pool_init(8 * 600)
    ptr, nb = dev.kv_pool_ptr()
    ppd.check(ppd.lib().ppd_op_fill_random(ptr, nb // 2, 7, 99, 0, None))
    rng = np.random.default_rng(0)
    only = os.environ.get("PPD_PROFILE_ONLY") == "1"

    def run(q_len, ctx, n=5, prof=False):
        nseq = len(q_len)
        maxb = max((c + q + 15) // 16 for q, c in zip(q_len, ctx))
        bt = np.arange(nseq * maxb, dtype=np.int32).reshape(nseq, maxb) % (8 * 600)
        toks = rng.integers(0, cfg.vocab, int(sum(q_len))).astype(np.int32)
        for _ in range(2):
            dev.step(q_len, ctx, toks, bt)
        if only:
            torch.cuda.profiler.start()
            dev.step(q_len, ctx, toks, bt)
            torch.cuda.profiler.stop()
            return None
        ms = float(np.median([dev.step(q_len, ctx, toks, bt).ms for _ in range(n)]))
        dev.set_profiling(True)
        dev.reset_stats()
        dev.step(q_len, ctx, toks, bt)
        st = dev.stats()
        dev.set_profiling(False)
        return {"q_len": q_len[:2] + (["..."] if len(q_len) > 2 else []), "n_seqs": nseq, "ctx": ctx[:2],
                "ms": ms, "pflops": flops(q_len, ctx) / (ms * 1e-3) / 1e15,
                "attn_ms": st["attn_ms"], "gemm_ms": st["gemm_ms"], "other_ms": st["step_ms"] - st["attn_ms"] - st["gemm_ms"]}

    if only:
        run([1536] + [1] * 8, [4096] + [1024] * 8)
        return
    for ctx in (2048, 4096, 6144):
        print(json.dumps({"case": "ppd_append_step", **run([1536] + [1] * 8, [ctx] + [1024] * 8)}), flush=True)
    for n in (3584, 5632, 7680):
        print(json.dumps({"case": "pd_full_prefill", **run([n], [0])}), flush=True)
    L = ppd.lib()
    from tools.gemm_sweep import t_us
    T = 1544
    for N, K in ((6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336)):
        A = torch.randn(T, K, device="cuda").to(torch.bfloat16)
        B = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
        C = torch.empty(2, T, N, device="cuda")
        m = torch.empty(T, N // 2, device="cuda", dtype=torch.bfloat16)
        f = 2.0 * T * N * K / 1e6
        res = {"case": "gemm", "T": T, "N": N, "K": K,
               "cublas_TF": f / t_us(lambda: L.ppd_op_gemm(A.data_ptr(), B.data_ptr(), C.data_ptr(), T, N, K, 1, None))}
        parts = ppd.GemmParts()
        res["tc_parts_TF"] = f / t_us(lambda: L.ppd_op_gemm_parts(A.data_ptr(), B.data_ptr(), C.data_ptr(), T, N, K, 2,
                                                                    parts, None))
        if N == 28672:
            res["tc_silu_TF"] = f / t_us(lambda: L.ppd_op_gemm_silu(A.data_ptr(), B.data_ptr(), m.data_ptr(), T, N, K,
                                                                     None))
        print(json.dumps({k: round(v, 1) if isinstance(v, float) else v for k, v in res.items()}), flush=True)
    dev.close()


if __name__ == "__main__":
    main()
