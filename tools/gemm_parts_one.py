"""Launch ppd_op_gemm_parts for ncu captures:
  PPD_ONE="T:N:K:pair:sched,..." python tools/gemm_parts_one.py
Each spec is launched 4 times over rotating weight copies (> L2)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_13358_b200 as ppd  # noqa: E402


def main():
    L = ppd.lib()
    for item in os.environ.get("PPD_ONE", "200:28672:4096:1:1").split(","):
        T, N, K, pair, sched = (int(x) for x in item.split(":"))
        ppd.check(L.ppd_set_tuning(b"gemm_pair", pair))
        ppd.check(L.ppd_set_tuning(b"gemm_sched", sched))
        A = torch.randn(T, K, device="cuda").to(torch.bfloat16)
        Ws = [(torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(2)]
        C = torch.empty(8, T, N, device="cuda")
        parts = ppd.GemmParts()
        for i in range(4):
            ppd.check(L.ppd_op_gemm_parts(A.data_ptr(), Ws[i % 2].data_ptr(), C.data_ptr(), T, N, K, 8,
                                          ctypes.byref(parts), None))
        torch.cuda.synchronize()
        print(item, "ok", parts.n, flush=True)


if __name__ == "__main__":
    main()
