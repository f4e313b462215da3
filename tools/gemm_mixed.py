"""Mixed-step GEMMs (decode rows + an append chunk: T = 200 ... 1736 token
rows) against their roofline max(weight bytes / HBM peak, 2TNK / tensor
peak), ours (ppd_op_gemm_parts auto plan; fused SiLU for gate|up) beside
cuBLAS, with ROTATING weight copies so every timed loop streams > L2 of
weights as inside a 32-layer step. CUDA events after warm-up.
  PPD_MIX_T="200,328,456" python tools/gemm_mixed.py"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_13358_b200 as ppd  # noqa: E402

HBM, TC = 6538e9, 1644.5e12


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
    ts = [int(x) for x in os.environ.get("PPD_MIX_T", "200,328,456,712,1224,1736").split(",")]
    knobs = [kv.split("=") for kv in filter(None, os.environ.get("PPD_MIX_KNOBS", "").split(","))]
    for k, v in knobs:
        ppd.check(L.ppd_set_tuning(k.encode(), int(v)))
    for N, K in ((6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336)):
        wbytes = N * K * 2
        ncopy = max(2, -(-400_000_000 // wbytes))
        Ws = [(torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16) for _ in range(ncopy)]
        for T in ts:
            A = torch.randn(T, K, device="cuda").to(torch.bfloat16)
            C = torch.empty(8, T, N, device="cuda")
            bound = max(wbytes / HBM, 2.0 * T * N * K / TC) * 1e6
            res = {"T": T, "N": N, "K": K, "bound_us": round(bound, 2)}
            parts = ppd.GemmParts()
            us = timed([(lambda W=W: L.ppd_op_gemm_parts(A.data_ptr(), W.data_ptr(), C.data_ptr(), T, N, K, 8,
                                                          ctypes.byref(parts), None)) for W in Ws])
            res.update(ours_us=round(us, 2), ours_frac=round(bound / us, 3), ours_slices=parts.n)
            us = timed([(lambda W=W: L.ppd_op_gemm(A.data_ptr(), W.data_ptr(), C.data_ptr(), T, N, K, 1, None))
                        for W in Ws])
            res.update(cublas_us=round(us, 2), cublas_frac=round(bound / us, 3))
            if N == 28672:
                M = torch.empty(T, N // 2, device="cuda", dtype=torch.bfloat16)
                us = timed([(lambda W=W: L.ppd_op_gemm_silu(A.data_ptr(), W.data_ptr(), M.data_ptr(), T, N, K, None))
                            for W in Ws])
                res.update(silu_us=round(us, 2), silu_frac=round(bound / us, 3))
            print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
