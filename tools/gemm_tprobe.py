"""Probe: decode-GEMM weight-streaming bandwidth vs token count T, for each
(kernel, schedule) choice of the fp32 forward path (ppd_op_gemm_parts):
single-CTA / CTA-pair kernel x uniform K split / balanced partition, and the
planner's automatic pick. CUDA events, after warm-up; weights > L2."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_13358_b200 as ppd  # noqa: E402
from tools.gemm_sweep import t_us  # noqa: E402

MODES = {"single-uniform": (0, 0), "pair-uniform": (1, 0), "single-balanced": (0, 1), "pair-balanced": (1, 1),
         "auto": (-1, -1)}


def main():
    L = ppd.lib()
    shapes = [(6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336), (128256, 4096)]
    ts = [int(x) for x in os.environ.get("PPD_TPROBE_T", "16,64,128,200,256").split(",")]
    for N, K in shapes:
        B = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
        for T in ts:
            A = torch.randn(T, K, device="cuda").to(torch.bfloat16)
            C = torch.empty(8, T, N, device="cuda")
            res = {"T": T, "N": N, "K": K}
            for name, (pair, sched) in MODES.items():
                ppd.check(L.ppd_set_tuning(b"gemm_pair", pair))
                ppd.check(L.ppd_set_tuning(b"gemm_sched", sched))
                parts = ppd.GemmParts()
                us = t_us(lambda: L.ppd_op_gemm_parts(A.data_ptr(), B.data_ptr(), C.data_ptr(), T, N, K, 8,
                                                      ctypes.byref(parts), None))
                res[name] = round(N * K * 2 / us / 1e6, 3)
                res[name + "_n"] = parts.n
            ppd.check(L.ppd_set_tuning(b"gemm_pair", -1))
            ppd.check(L.ppd_set_tuning(b"gemm_sched", -1))
            print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
