"""Prefill-size GEMMs (T = 1736: a 1536-token append + 200 decode rows, and
2048 / 4096): tcgen05 kernel (uniform K splits 1/2, fused SiLU for gate|up) vs
cuBLAS, CUDA events after warm-up; TFLOP/s = 2 T N K / time."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_13358_b200 as ppd  # noqa: E402
from tools.gemm_sweep import t_us  # noqa: E402


def main():
    L = ppd.lib()
    for T in (1736, 2048, 4096):
        for N, K in ((6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336)):
            A = torch.randn(T, K, device="cuda").to(torch.bfloat16)
            B = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
            C = torch.empty(2, T, N, device="cuda")
            m = torch.empty(T, N // 2, device="cuda", dtype=torch.bfloat16)
            f = 2.0 * T * N * K / 1e6
            res = {"T": T, "N": N, "K": K,
                   "cublas_TF": f / t_us(lambda: L.ppd_op_gemm(A.data_ptr(), B.data_ptr(), C.data_ptr(), T, N, K, 1, None))}
            for sp in (1, 2):
                res[f"tc_s{sp}_TF"] = f / t_us(lambda: L.ppd_op_gemm_tc(A.data_ptr(), B.data_ptr(), C.data_ptr(), T, N,
                                                                         K, 1, sp, None))
            if N == 28672:
                res["tc_silu_TF"] = f / t_us(lambda: L.ppd_op_gemm_silu(A.data_ptr(), B.data_ptr(), m.data_ptr(), T, N,
                                                                         K, None))
            print(json.dumps({k: round(v, 1) if isinstance(v, float) else v for k, v in res.items()}), flush=True)


if __name__ == "__main__":
    main()
