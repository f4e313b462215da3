"""Prefill-shape GEMM A/B of tuning knobs in one process (alternating):
  PPD_PK="gemm_multi_sub" PPD_PK_T=1546,2058,4096 python tools/gemm_pf_knob.py"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_13358_b200 as ppd  # noqa: E402
from tools.gemm_sweep import t_us  # noqa: E402


def main():
    L = ppd.lib()
    knob = os.environ.get("PPD_PK", "gemm_multi_sub").encode()
    for T in (int(x) for x in os.environ.get("PPD_PK_T", "1546,2058,4096").split(",")):
        for N, K in ((6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336)):
            A = torch.randn(T, K, device="cuda").to(torch.bfloat16)
            B = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
            C = torch.empty(2, T, N, device="cuda")
            parts = ppd.GemmParts()
            res = {0: [], 1: []}
            for _ in range(4):
                for v in (0, 1):
                    ppd.check(L.ppd_set_tuning(knob, v))
                    res[v].append(t_us(lambda: L.ppd_op_gemm_parts(A.data_ptr(), B.data_ptr(), C.data_ptr(), T, N, K,
                                                                   1, ppd.ctypes.byref(parts), None), iters=10))
            ppd.check(L.ppd_set_tuning(knob, 0))
            out = {"T": T, "N": N, "K": K}
            for v in (0, 1):
                us = float(np.median(res[v]))
                out[f"{knob.decode()}={v}_TFs"] = round(2 * T * N * K / us / 1e6, 1)
            print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
