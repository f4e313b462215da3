"""K5 parity: the tcgen05/TMEM/TMA GEMM (gemm_tc.cu) against the cuBLAS library
GEMM and an fp32 torch reference, on the shapes the forward step uses
(decode: <=256 token rows, weight-streaming with K-split partials; prefill:
many token tiles), plus ragged token counts. Tolerance (stated): fp32 output
within 1e-3 * sqrt(K) * max|ref| of the fp32 reference (different summation
order only); bf16 output within 1 bf16 ulp of the rounded reference."""
import ctypes

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


@pytest.fixture(params=[0, 1], ids=["single", "pair"])
def pair_mode(request):
    ppd.check(ppd.lib().ppd_set_tuning(b"gemm_pair", request.param))
    yield request.param
    ppd.check(ppd.lib().ppd_set_tuning(b"gemm_pair", -1))


@pytest.mark.parametrize("M,N,K,splits", [
    (200, 6144, 4096, 3),     # decode QKV (Llama-8B), K-split
    (200, 4096, 14336, 4),    # decode down-proj
    (200, 28672, 4096, 1),    # decode gate|up
    (37, 768, 512, 1),        # tiny model, ragged token count
    (1, 2048, 512, 1),        # single row
    (1224, 6144, 4096, 1),    # decode + one 1024-token prefill chunk
    (777, 1000, 256, 2),      # ragged N and M
    (5, 128256, 4096, 1),     # lm_head of a few rows
    (4096, 6144, 4096, 1),    # prefill QKV, 16 token tiles
    (200, 300, 4096, 3),      # weight rows not a multiple of the 256-row pair tile
    (328, 28672, 4096, 1),    # decode + 128-token append chunk: one unit, 2 token sub-tiles
    (300, 6144, 4096, 3),     # 2 sub-tiles with K split
    (512, 4096, 4096, 2),     # largest 2-sub-tile step
    (257, 768, 512, 1),       # one row past a single tile, tiny model
])
def test_gemm_tc_fp32(gpu, pair_mode, M, N, K, splits):
    run(M, N, K, splits)


def test_gemm_tc_bf16_out(gpu, pair_mode):
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


def test_gemm_pair_equals_single(gpu):
    """Both kernels accumulate each output in the same K order per split, so the
    CTA-pair path must reproduce the single-CTA result bit for bit."""
    import torch
    M, N, K = 200, 6144, 4096
    A = (torch.randn(M, K, device="cuda") * 0.5).to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    outs = []
    L = ppd.lib()
    try:
        for mode in (0, 1):
            ppd.check(L.ppd_set_tuning(b"gemm_pair", mode))
            C = torch.zeros(3, M, N, device="cuda")
            ppd.check(L.ppd_op_gemm_tc(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, 1, 3, None))
            outs.append(C)
    finally:
        ppd.check(L.ppd_set_tuning(b"gemm_pair", -1))
    assert torch.equal(outs[0], outs[1])


def test_l2_hint_does_not_change_results(gpu):
    """The L2 evict-first policy on the weight stream (knob l2_hint) is a cache
    hint only: results are bit-identical with and without it."""
    import torch
    M, N, K = 200, 6144, 4096
    A = (torch.randn(M, K, device="cuda") * 0.5).to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    outs = []
    L = ppd.lib()
    try:
        for mask in (0, 3):
            ppd.check(L.ppd_set_tuning(b"l2_hint", mask))
            C = torch.zeros(3, M, N, device="cuda")
            ppd.check(L.ppd_op_gemm_tc(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, 1, 3, None))
            outs.append(C)
        with pytest.raises(ppd.InvalidArgument):
            ppd.check(L.ppd_set_tuning(b"l2_hint", 4))
    finally:
        ppd.check(L.ppd_set_tuning(b"l2_hint", 3))
    assert torch.equal(outs[0], outs[1])


def test_set_tuning_rejects_unknown(gpu):
    with pytest.raises(ppd.InvalidArgument):
        ppd.check(ppd.lib().ppd_set_tuning(b"no_such_knob", 1))


@pytest.fixture(params=[(0, 1), (1, 1), (1, 0)], ids=["single-balanced", "pair-balanced", "pair-uniform"])
def sched_mode(request):
    pair, sched = request.param
    L = ppd.lib()
    ppd.check(L.ppd_set_tuning(b"gemm_pair", pair))
    ppd.check(L.ppd_set_tuning(b"gemm_sched", sched))
    yield request.param
    ppd.check(L.ppd_set_tuning(b"gemm_pair", -1))
    ppd.check(L.ppd_set_tuning(b"gemm_sched", -1))


@pytest.mark.parametrize("M,N,K", [
    (200, 28672, 4096),   # decode gate|up: 224 / 112 tiles do not divide the SMs
    (200, 4096, 14336),   # decode down-proj
    (200, 6144, 4096),    # decode QKV
    (37, 768, 512),       # tiny model
    (1224, 6144, 4096),   # decode + prefill chunk: several token tiles
    (200, 300, 4096),     # ragged weight rows
    (328, 28672, 4096),   # decode + append chunk: 2 token sub-tiles per unit
    (456, 4096, 14336),   # 2 sub-tiles, long K
    (2048, 4096, 14336),  # prefill: whole waves + stream-K tail
    (1736, 4096, 4096),   # prefill: whole waves + stream-K tail, short K
])
def test_gemm_parts_partition(gpu, sched_mode, M, N, K):
    """The fp32 path the forward step uses: only the slices GemmParts marks
    valid are summed (the rest stay NaN-poisoned), and the sum equals A.B^T."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(1)
    A = (torch.randn(M, K, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    ref = A.float() @ B.float().t()
    max_sl = 8
    C = torch.full((max_sl, M, N), float("nan"), device="cuda")
    parts = ppd.GemmParts()
    ppd.check(ppd.lib().ppd_op_gemm_parts(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, max_sl,
                                          ctypes.byref(parts), None))
    torch.cuda.synchronize()
    assert 1 <= parts.n <= max_sl and parts.stride == M * N
    col = torch.arange(N, device="cuda").view(1, N)
    tok = torch.arange(M, device="cuda").view(M, 1)
    nvalid = parts.valid(col, tok)
    got = torch.zeros(M, N, device="cuda")
    for j in range(parts.n):
        got += torch.where(nvalid > j, C[j], torch.zeros_like(got))
    assert torch.isfinite(got).all(), "a valid slice was not written"
    tol = 1e-3 * np.sqrt(K) * ref.abs().max().item()
    assert (got - ref).abs().max().item() <= tol


@pytest.mark.parametrize("M,N,K", [(200, 28672, 4096), (37, 2048, 512), (1224, 28672, 4096), (5, 384, 512),
                                   (328, 28672, 4096), (300, 384, 512)])
def test_gemm_silu_fused(gpu, pair_mode, M, N, K):
    """Fused SiLU epilogue vs fp32 torch of the interleaved gate|up layout:
    m = bf16(silu(g) * u), within 1 bf16 ulp (+ the fp32 GEMM tolerance)."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(2)
    A = (torch.randn(M, K, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    m = torch.full((M, N // 2), float("nan"), device="cuda").to(torch.bfloat16)
    ppd.check(ppd.lib().ppd_op_gemm_silu(A.data_ptr(), B.data_ptr(), m.data_ptr(), M, N, K, None))
    torch.cuda.synchronize()
    y = (A.float() @ B.float().t()).view(M, N // 128, 2, 64)
    gate, up = y[:, :, 0, :].reshape(M, N // 2), y[:, :, 1, :].reshape(M, N // 2)
    ref = gate / (1.0 + torch.exp(-gate)) * up
    got = m.float()
    assert torch.isfinite(got).all()
    tol = 2 ** -7 * ref.abs() + 1e-3 * np.sqrt(K) * ref.abs().max().item()
    assert ((got - ref).abs() <= tol).all()
