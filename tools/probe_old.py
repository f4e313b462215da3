import ctypes, os, sys, torch
lib = ctypes.CDLL(sys.argv[1])
vp, i32 = ctypes.c_void_p, ctypes.c_int32
has_tc = hasattr(lib, "ppd_op_gemm_tc")
def t_us(fn, iters=30):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / iters * 1e3
for N, K in ((28672, 4096), (6144, 4096)):
    T = 200
    A = torch.randn(T, K, device="cuda").to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    C = torch.empty(4, T, N, device="cuda")
    lib.ppd_op_gemm_tc.argtypes = [vp, vp, vp, i32, i32, i32, i32, i32, vp]
    for sp in (1, 3):
        print(sys.argv[1].split('/')[-2], N, sp, round(t_us(lambda: lib.ppd_op_gemm_tc(A.data_ptr(), B.data_ptr(), C.data_ptr(), T, N, K, 1, sp, None)), 1), flush=True)
