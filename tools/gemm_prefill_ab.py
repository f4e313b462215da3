"""Prefill-shape GEMMs (T = 1024..4096 token rows): single-CTA vs CTA-pair
tcgen05 kernel, fp32 output (uniform, no K split). TFLOP/s by CUDA events."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_13358_b200 as ppd  # noqa: E402
from tools.gemm_sweep import t_us  # noqa: E402


def main():
    L = ppd.lib()
    Ts = [int(x) for x in os.environ.get("PPD_PF_T", "1024,1224,2048,4096").split(",")]
    for T in Ts:
        for N, K in ((6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336)):
            A = torch.randn(T, K, device="cuda").to(torch.bfloat16)
            B = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
            C = torch.empty(T, N, device="cuda")
            res = {"T": T, "N": N, "K": K}
            for pair in (0, 1):
                ppd.check(L.ppd_set_tuning(b"gemm_pair", pair))
                us = t_us(lambda: L.ppd_op_gemm_tc(A.data_ptr(), B.data_ptr(), C.data_ptr(), T, N, K, 1, 1, None))
                res[f"pair{pair}_TFs"] = round(2 * T * N * K / us / 1e6, 1)
            us = t_us(lambda: L.ppd_op_gemm(A.data_ptr(), B.data_ptr(), C.data_ptr(), T, N, K, 1, None))
            res["cublas_TFs"] = round(2 * T * N * K / us / 1e6, 1)
            ppd.check(L.ppd_set_tuning(b"gemm_pair", -1))
            print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
