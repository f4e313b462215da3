"""In-process A/B of the decode-shape GEMMs between two builds of libppd_b200.so
(e.g. a commit in old_build/<sha>/ vs the working tree): launches alternate
between the libraries round by round so clock / power drift hits both alike.

  python tools/ab_libs.py old_build/<sha>/paper_2603_13358_b200/libppd_b200.so \
      paper_2603_13358_b200/libppd_b200.so
Per library, optional tuning after a colon: path:gemm_pair=0,gemm_sched=0
"""
import ctypes
import json
import sys

import numpy as np
import torch


def load(spec):
    path, _, kv = spec.partition(":")
    lib = ctypes.CDLL(path)
    vp, i32 = ctypes.c_void_p, ctypes.c_int32
    lib.ppd_op_gemm_tc.argtypes = [vp, vp, vp, i32, i32, i32, i32, i32, vp]
    tun = {}
    for pair in filter(None, kv.split(",")):
        k, v = pair.split("=")
        tun[k] = int(v)
    if tun:
        lib.ppd_set_tuning.argtypes = [ctypes.c_char_p, i32]
        for k, v in tun.items():
            assert lib.ppd_set_tuning(k.encode(), v) == 0, k
    return spec, lib


def t_us(fn, iters=20):
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
    libs = [load(s) for s in sys.argv[1:]]
    import os
    T = int(os.environ.get("PPD_AB_T", "200"))
    shapes = [(6144, 4096, 3), (4096, 4096, 4), (28672, 4096, 1), (4096, 14336, 4), (128256, 4096, 1)]
    if T > 512:  # prefill shapes: no K split
        shapes = [(6144, 4096, 1), (4096, 4096, 1), (28672, 4096, 1), (4096, 14336, 1)]
    for N, K, sp in shapes:
        A = torch.randn(T, K, device="cuda").to(torch.bfloat16)
        B = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
        C = torch.empty(8, T, N, device="cuda")
        res = {name: [] for name, _ in libs}
        for _ in range(6):
            for name, lib in libs:
                res[name].append(t_us(lambda: lib.ppd_op_gemm_tc(A.data_ptr(), B.data_ptr(), C.data_ptr(), T, N, K,
                                                                  1, sp, None)))
        out = {"N": N, "K": K, "splits": sp}
        for i, (name, _) in enumerate(libs):
            out[f"lib{i}_us"] = round(float(np.median(res[name])), 2)
            out[f"lib{i}_TBs"] = round(N * K * 2 / np.median(res[name]) / 1e6, 2)
            out[f"lib{i}_TFs"] = round(2 * T * N * K / np.median(res[name]) / 1e6, 1)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
