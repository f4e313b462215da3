"""Launch one decode-shape GEMM 3x through a given libppd_b200.so (for ncu):
  python tools/one_gemm_lib.py <lib.so>[:knob=v,...] N K splits"""
import ctypes
import sys

import torch

spec, N, K, sp = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
path, _, kv = spec.partition(":")
lib = ctypes.CDLL(path)
vp, i32 = ctypes.c_void_p, ctypes.c_int32
lib.ppd_op_gemm_tc.argtypes = [vp, vp, vp, i32, i32, i32, i32, i32, vp]
for pair in filter(None, kv.split(",")):
    k, v = pair.split("=")
    lib.ppd_set_tuning.argtypes = [ctypes.c_char_p, i32]
    assert lib.ppd_set_tuning(k.encode(), int(v)) == 0
import os
T = int(os.environ.get("PPD_ONE_T", "200"))
A = torch.randn(T, K, device="cuda").to(torch.bfloat16)
B = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
C = torch.empty(sp, T, N, device="cuda")
for _ in range(3):
    lib.ppd_op_gemm_tc(A.data_ptr(), B.data_ptr(), C.data_ptr(), T, N, K, 1, sp, None)
torch.cuda.synchronize()
