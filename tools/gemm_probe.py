"""Probe the decode GEMM bottleneck: same weights (N x K), varying token count T
(activation bytes per stage) and K-split, tcgen05 kernel only."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_13358_b200 as ppd  # noqa: E402


def t_us(fn, iters=30):
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


N, K = int(os.environ.get("PN", 28672)), int(os.environ.get("PK", 4096))
B = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
for T in (16, 64, 128, 200, 256):
    A = torch.randn(T, K, device="cuda").to(torch.bfloat16)
    C = torch.empty(4, T, N, device="cuda")
    L = ppd.lib()
    row = [T]
    for sp in (0, 1, 2):
        us = t_us(lambda: L.ppd_op_gemm_tc(A.data_ptr(), B.data_ptr(), C.data_ptr(), T, N, K, 1, sp, None))
        row.append(f"s{sp}={us:.1f}us {N*K*2/us/1e6:.2f}TB/s")
    print(os.environ.get("PPD_GEMM_STAGES", "auto"), row, flush=True)
