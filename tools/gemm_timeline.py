"""Per-CTA timeline of one decode-shape tcgen05 GEMM (gemm_diag bit 2,
globaltimer): setup, first-data latency, main loop, epilogue tail.
  PPD_TL="200:28672:4096,200:4096:14336" python tools/gemm_timeline.py"""
import ctypes
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_13358_b200 as ppd  # noqa: E402


def main():
    L = ppd.lib()
    ppd.check(L.ppd_set_tuning(b"ops_w_tiled", 1))
    for item in os.environ.get("PPD_TL", "200:28672:4096,200:4096:14336,200:6144:4096,328:28672:4096").split(","):
        T, N, K = (int(x) for x in item.split(":"))
        Ws = []
        for _ in range(3):
            W = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
            Wt = torch.empty_like(W)
            ppd.check(L.ppd_op_tile_matrix(W.data_ptr(), Wt.data_ptr(), N, K, None))
            Ws.append(Wt)
        A = torch.randn(T, K, device="cuda").to(torch.bfloat16)
        C = torch.empty(8, T, N, device="cuda")
        parts = ppd.GemmParts()
        for i in range(6):
            ppd.check(L.ppd_op_gemm_parts(A.data_ptr(), Ws[i % 3].data_ptr(), C.data_ptr(), T, N, K, 8,
                                          ctypes.byref(parts), None))
        torch.cuda.synchronize()
        for mode in ("isolated", "pdl_chain"):
            ppd.check(L.ppd_set_tuning(b"gemm_diag", 4))
            if mode == "pdl_chain":  # previous GEMM still running when this one launches
                ppd.check(L.ppd_op_gemm_parts(A.data_ptr(), Ws[1].data_ptr(), C.data_ptr(), T, N, K, 8,
                                              ctypes.byref(parts), None))
            ppd.check(L.ppd_op_gemm_parts(A.data_ptr(), Ws[2].data_ptr(), C.data_ptr(), T, N, K, 8,
                                          ctypes.byref(parts), None))
            torch.cuda.synchronize()
            ppd.check(L.ppd_set_tuning(b"gemm_diag", 0))
            buf = (ctypes.c_uint64 * (512 * 6))()
            n = L.ppd_op_gemm_timeline(buf, 512)
            a = np.frombuffer(buf, dtype=np.uint64).reshape(512, 6)[:n].astype(np.int64)
            a = a[a[:, 0] > 0]
            # only rows written by this launch: the most recent entry stamps
            t0 = a[:, 0].max() - 200_000
            a = a[a[:, 0] >= t0]
            base = a[:, 0].min()
            rel = (a - base) / 1e3  # us
            mma = a[a[:, 3] > 0]
            q = lambda v: [round(float(np.min(v)), 2), round(float(np.median(v)), 2), round(float(np.max(v)), 2)]
            res = {"T": T, "N": N, "K": K, "mode": mode, "ctas": int(len(a)), "slices": parts.n,
                   "span_us": round(float((a[:, 5].max() - base) / 1e3), 2),
                   "entry_us": q(rel[:, 0]), "setup_us": q((a[:, 1] - a[:, 0]) / 1e3),
                   "first_data_us": q((mma[:, 2] - mma[:, 1]) / 1e3),
                   "main_us": q((mma[:, 3] - mma[:, 2]) / 1e3),
                   "main_end_rel_us": q((mma[:, 3] - base) / 1e3),
                   "epi_tail_us": q((a[:, 4] - a[:, 3].clip(min=1)) / 1e3) if len(mma) == len(a) else None,
                   "exit_rel_us": q(rel[:, 5]),
                   "w_gbs_main": round(N * K * 2 / (float(np.median(mma[:, 3] - mma[:, 2])) / 1e9) / 1e9, 1)}
            print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
