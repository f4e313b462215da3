"""Decode-GEMM sensitivity probe: weight-streaming TB/s of the fp32 forward
path (ppd_op_gemm_parts, tiled weights rotating over > L2) under tuning knobs
and timing-only diagnostics (gemm_diag: 1 skip activation loads, 2 skip MMAs).
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
    {}, {"gemm_occ2": 0}, {"gemm_occ2": 1, "gemm_pair": 0}, {"gemm_occ2": 1, "gemm_pair": 0, "gemm_sched": 1},
    {"gemm_occ2": 0, "gemm_pair": 0}, {"gemm_occ2": 0, "gemm_pair": 1},
]
if os.environ.get("PPD_KN_WS"):
    VARIANTS = [{}, {"gemm_wsplit": 2}, {"gemm_wsplit": 4}, {"gemm_wsplit": 8},
    {"gemm_diag": 3}, {"gemm_wsplit": 2, "gemm_diag": 3}, {"gemm_wsplit": 4, "gemm_diag": 3},
    {"gemm_wsplit": 8, "gemm_diag": 3},
    {"gemm_pair": 0}, {"gemm_pair": 0, "gemm_wsplit": 4}, {"gemm_pair": 1, "gemm_wsplit": 4},
    {"gemm_stages": 4, "gemm_wsplit": 4},
]
if os.environ.get("PPD_KN_OLD"):
    VARIANTS = [
        {}, {"gemm_stages": 3}, {"gemm_stages": 4}, {"gemm_stages": 5},
        {"gemm_w_promo": 0}, {"gemm_w_promo": 1},
        {"gemm_diag": 1}, {"gemm_diag": 2}, {"gemm_diag": 3},
        {"gemm_pair": 0}, {"gemm_pair": 1}, {"gemm_pair": 0, "gemm_diag": 1}, {"gemm_pair": 0, "gemm_diag": 3},
        {"gemm_sched": 0}, {"gemm_sched": 1},
    ]
DEFAULTS = {"gemm_occ2": -1, "gemm_stages": 0, "gemm_w_promo": 2, "gemm_diag": 0, "gemm_pair": -1, "gemm_sched": -1,
            "gemm_wsplit": 1}


def main():
    L = ppd.lib()
    ts = [int(x) for x in os.environ.get("PPD_KN_T", "200").split(",")]
    shapes = [(28672, 4096), (4096, 14336), (6144, 4096)]
    ppd.check(L.ppd_set_tuning(b"ops_w_tiled", 1))
    for N, K in shapes:
        wbytes = N * K * 2
        ncopy = max(2, -(-400_000_000 // wbytes))
        Ws = []
        for _ in range(ncopy):
            W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
            Wt = torch.empty_like(W)
            ppd.check(L.ppd_op_tile_matrix(W.data_ptr(), Wt.data_ptr(), N, K, None))
            Ws.append(Wt)
            del W
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
