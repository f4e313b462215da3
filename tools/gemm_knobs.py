"""Decode-GEMM sensitivity probe: weight-streaming TB/s of the fp32 forward
path (ppd_op_gemm_parts, weights rotating over > L2) under the tuning knobs.
  PPD_KN_T=200 python tools/gemm_knobs.py"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_13358_b200 as ppd  # noqa: E402
from tools.gemm_rot import timed  # noqa: E402

VARIANTS = [
    {}, {"gemm_occ2": 0}, {"gemm_occ2": 1, "gemm_pair": 0}, {"gemm_multi_sub": 0},
    {"gemm_pair": 0}, {"gemm_pair": 1}, {"gemm_sched": 0}, {"gemm_sched": 1},
]
DEFAULTS = {"gemm_occ2": 0, "gemm_stages": 0, "gemm_pair": -1, "gemm_sched": -1, "gemm_multi_sub": 1}


def main():
    L = ppd.lib()
    ts = [int(x) for x in os.environ.get("PPD_KN_T", "200").split(",")]
    shapes = [(28672, 4096), (4096, 14336), (6144, 4096)]
    for N, K in shapes:
        wbytes = N * K * 2
        ncopy = max(2, -(-400_000_000 // wbytes))
        Ws = [(torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(ncopy)]
        for T in ts:
            A = torch.randn(T, K, device="cuda").to(torch.bfloat16)
            C = torch.empty(8, T, N, device="cuda")
            res = {"T": T, "N": N, "K": K}
            for v in VARIANTS:
                for k, x in v.items():
                    ppd.check(L.ppd_set_tuning(k.encode(), x))
                parts = ppd.GemmParts()
                fns = [(lambda W=W: L.ppd_op_gemm_parts(A.data_ptr(), W.data_ptr(), C.data_ptr(), T, N, K, 8,
                                                        ctypes.byref(parts), None)) for W in Ws]
                us = timed(fns)
                res[",".join(f"{k}={x}" for k, x in v.items()) or "base"] = round(wbytes / us / 1e6, 3)
                for k in v:
                    ppd.check(L.ppd_set_tuning(k.encode(), DEFAULTS[k]))
            print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
