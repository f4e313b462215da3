"""Launch one tcgen05 GEMM per (T, pair mode) for an ncu capture:
  PPD_ONE="T:N:K:splits:pair,..." python tools/gemm_one.py
Each shape is launched 3 times (ncu -c/-s pick which); splits 0 = the fused
SiLU gate|up GEMM."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_13358_b200 as ppd  # noqa: E402


def main():
    L = ppd.lib()
    spec = os.environ.get("PPD_ONE", "16:28672:4096:1:1,200:28672:4096:1:1,200:28672:4096:1:0")
    for item in spec.split(","):
        T, N, K, sp, pair = (int(x) for x in item.split(":"))
        ppd.check(L.ppd_set_tuning(b"gemm_pair", pair))
        A = torch.randn(T, K, device="cuda").to(torch.bfloat16)
        B = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
        C = torch.empty(max(sp, 1), T, N, device="cuda")
        m = torch.empty(T, N // 2, device="cuda", dtype=torch.bfloat16)
        for _ in range(3):
            if sp == 0:  # fused SiLU gate|up epilogue (bf16 m out)
                ppd.check(L.ppd_op_gemm_silu(A.data_ptr(), B.data_ptr(), m.data_ptr(), T, N, K, None))
            else:
                ppd.check(L.ppd_op_gemm_tc(A.data_ptr(), B.data_ptr(), C.data_ptr(), T, N, K, 1, sp, None))
        torch.cuda.synchronize()
        print(item, "ok", flush=True)


if __name__ == "__main__":
    main()
