"""3xTF32 GEMM accuracy vs K (fp64 reference) next to torch fp32 matmul: shows the per-k-block
chunked accumulation keeps the error independent of K."""
import ctypes, sys, torch
sys.path.insert(0, "/root/repo")
from paper_2105_04779_b200 import capi
L = capi.lib()
vp, i32, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
L.elattn_gpu_testing_gemm_tf32x3.argtypes = [vp, i64, i64, vp, i64, i64, vp, vp, i64, i64, vp, i64, i32, i32, i32, i32, ctypes.c_float, vp]
for K in (64, 128, 256, 512, 1024, 2048, 4096):
    M, N, Z = 256, 256, 1
    g = torch.Generator(device="cuda").manual_seed(K)
    A = torch.rand(Z, M, K, generator=g, device="cuda") * 2 - 1
    B = torch.rand(Z, N, K, generator=g, device="cuda") * 2 - 1
    C = torch.zeros(Z, M, N, device="cuda")
    capi.check(L.elattn_gpu_testing_gemm_tf32x3(A.data_ptr(), K, M*K, B.data_ptr(), K, N*K, C.data_ptr(), None, N, M*N, None, N, M, N, K, Z, 1.0, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    want = torch.einsum("zmk,znk->zmn", A.double(), B.double())
    f32 = torch.einsum("zmk,znk->zmn", A, B)  # torch fp32 (TF32 off by default for matmul? check)
    torch.backends.cuda.matmul.allow_tf32 = False
    f32b = torch.matmul(A, B.transpose(1, 2))
    e = lambda x: ((x.double() - want).abs().max() / want.abs().max()).item()
    # simulated fp32 sequential accumulation error bound
    print(K, "3xtf32 %.2e" % e(C), "torch-fp32 %.2e" % e(f32b), "mean|err| %.2e" % ((C.double()-want).abs().mean()/want.abs().mean()).item())
