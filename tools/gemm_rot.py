"""Decode-GEMM weight-streaming probe with ROTATING weight copies (the working
set of every timed loop is > L2, as inside a 32-layer step), per
(kernel, schedule) mode of the fp32 forward path (ppd_op_gemm_parts) and the
fused SiLU path. CUDA events on the launching stream, after warm-up.
  PPD_ROT_T="200,328" python tools/gemm_rot.py"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_13358_b200 as ppd  # noqa: E402

MODES = {"single-uniform": (0, 0), "pair-uniform": (1, 0), "single-balanced": (0, 1), "pair-balanced": (1, 1),
         "auto": (-1, -1)}


def timed(fns, iters=24):
    for f in fns[:3]:
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(iters):
        fns[i % len(fns)]()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters * 1e3


def main():
    L = ppd.lib()
    shapes = [(6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336)]
    ts = [int(x) for x in os.environ.get("PPD_ROT_T", "200,328").split(",")]
    modes = os.environ.get("PPD_ROT_MODES", ",".join(MODES)).split(",")
    for N, K in shapes:
        wbytes = N * K * 2
        ncopy = max(2, -(-400_000_000 // wbytes))
        Ws = [(torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(ncopy)]
        for T in ts:
            A = torch.randn(T, K, device="cuda").to(torch.bfloat16)
            C = torch.empty(8, T, N, device="cuda")
            res = {"T": T, "N": N, "K": K}
            for name in modes:
                pair, sched = MODES[name]
                ppd.check(L.ppd_set_tuning(b"gemm_pair", pair))
                ppd.check(L.ppd_set_tuning(b"gemm_sched", sched))
                parts = ppd.GemmParts()
                fns = [(lambda W=W: L.ppd_op_gemm_parts(A.data_ptr(), W.data_ptr(), C.data_ptr(), T, N, K, 8,
                                                        ctypes.byref(parts), None)) for W in Ws]
                us = timed(fns)
                res[name] = round(us, 2)
                res[name + "_tbs"] = round(wbytes / us / 1e6, 3)
                res[name + "_n"] = parts.n
            if N == 28672:
                for pair in (0, 1, -1):
                    ppd.check(L.ppd_set_tuning(b"gemm_pair", pair))
                    M = torch.empty(T, N // 2, device="cuda", dtype=torch.bfloat16)
                    fns = [(lambda W=W: L.ppd_op_gemm_silu(A.data_ptr(), W.data_ptr(), M.data_ptr(), T, N, K, None))
                           for W in Ws]
                    us = timed(fns)
                    res[f"silu_pair{pair}"] = round(us, 2)
                    res[f"silu_pair{pair}_tbs"] = round(wbytes / us / 1e6, 3)
            ppd.check(L.ppd_set_tuning(b"gemm_pair", -1))
            ppd.check(L.ppd_set_tuning(b"gemm_sched", -1))
            print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
