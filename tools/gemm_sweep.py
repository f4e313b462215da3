"""GEMM sweep on the GPU: tcgen05 kernel (ppd_op_gemm_tc) vs cuBLAS for the
forward step's shapes; CUDA events on the launching stream, after warm-up."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_13358_b200 as ppd  # noqa: E402

SHAPES = [(200, 6144, 4096), (200, 4096, 4096), (200, 28672, 4096), (200, 4096, 14336), (200, 128256, 4096),
          (4096, 6144, 4096), (4096, 28672, 4096), (4096, 4096, 14336)]


def t_us(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters * 1e3


def main():
    out = []
    for M, N, K in SHAPES:
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        B = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
        C = torch.empty(8, M, N, device="cuda")
        L = ppd.lib()
        res = {"M": M, "N": N, "K": K}
        res["cublas_us"] = t_us(lambda: L.ppd_op_gemm(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, 1, None))
        for sp in (1, 2, 3, 4, 6, 8):
            if (K // 64) // sp < 4:
                continue
            res[f"tc_s{sp}_us"] = t_us(lambda: L.ppd_op_gemm_tc(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K,
                                                                 1, sp, None))
        wbytes = N * K * 2
        best = min(v for k, v in res.items() if k.startswith("tc_"))
        res["best_tc_TBs"] = wbytes / best / 1e6
        res["cublas_TBs"] = wbytes / res["cublas_us"] / 1e6
        res["best_tc_TFs"] = 2 * M * N * K / best / 1e6
        out.append(res)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
