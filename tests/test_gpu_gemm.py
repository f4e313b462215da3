"""K5 parity: the tcgen05/TMEM/TMA GEMM (gemm_tc.cu) against the cuBLAS library
GEMM and an fp32 torch reference, on the shapes the forward step uses
(decode: <=256 token rows, weight-streaming with K-split partials; prefill:
many token tiles), plus ragged token counts. Tolerance (stated): fp32 output
within 1e-3 * sqrt(K) * max|ref| of the fp32 reference (different summation
order only); bf16 output within 1 bf16 ulp of the rounded reference."""
import numpy as np
import pytest

import paper_2603_13358_b200 as ppd

pytestmark = pytest.mark.gpu


def run(M, N, K, splits=1, out_f32=True, seed=0):
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    A = (torch.randn(M, K, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    ref = A.float() @ B.float().t()
    if out_f32:
        C = torch.zeros(max(splits, 1), M, N, device="cuda", dtype=torch.float32)
    else:
        C = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    ppd.check(ppd.lib().ppd_op_gemm_tc(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, 1 if out_f32 else 0,
                                       splits, None))
    got = C.sum(0) if out_f32 else C.float()
    tol = 1e-3 * np.sqrt(K) * ref.abs().max().item()
    err = (got - ref).abs().max().item()
    assert torch.isfinite(got).all()
    assert err <= (tol if out_f32 else 2 ** -7 * ref.abs().max().item()), (M, N, K, splits, err, tol)
    return got, ref


@pytest.mark.parametrize("M,N,K,splits", [
    (200, 6144, 4096, 3),     # decode QKV (Llama-8B), K-split
    (200, 4096, 14336, 4),    # decode down-proj
    (200, 28672, 4096, 1),    # decode gate|up
    (37, 768, 512, 1),        # tiny model, ragged token count
    (1, 2048, 512, 1),        # single row
    (1224, 6144, 4096, 1),    # decode + one 1024-token prefill chunk
    (777, 1000, 256, 2),      # ragged N and M
    (5, 128256, 4096, 1),     # lm_head of a few rows
])
def test_gemm_tc_fp32(gpu, M, N, K, splits):
    run(M, N, K, splits)


def test_gemm_tc_bf16_out(gpu):
    run(300, 4096, 4096, 1, out_f32=False)


def test_gemm_tc_matches_cublas(gpu):
    import torch
    M, N, K = 256, 4096, 4096
    A = (torch.randn(M, K, device="cuda") * 0.5).to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    C1 = torch.zeros(M, N, device="cuda")
    C2 = torch.zeros(M, N, device="cuda")
    ppd.check(ppd.lib().ppd_op_gemm_tc(A.data_ptr(), B.data_ptr(), C1.data_ptr(), M, N, K, 1, 1, None))
    ppd.check(ppd.lib().ppd_op_gemm(A.data_ptr(), B.data_ptr(), C2.data_ptr(), M, N, K, 1, None))
    assert (C1 - C2).abs().max().item() <= 1e-3 * C2.abs().max().item()
