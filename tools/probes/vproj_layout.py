import ctypes, json, sys
sys.path.insert(0, '/root/repo')
sys.path.insert(0, '.')
import torch
from paper_2105_04779_b200 import capi
L = capi.lib()
vp, i32, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
L.elattn_gpu_testing_gemm_bf16.argtypes = [vp, i64, i64, vp, i64, i64, vp, i64, i64, vp, i64, i32, i32, i32, i32, ctypes.c_float, i32, vp]
h, d_m, d_k = 16, 1024, 64
def graph_time(fn, reps=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps): fn()
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); g.replay(); e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
for B in (32, 320):
    R = B * 4
    C = torch.randn(R * h, d_m, device='cuda').to(torch.bfloat16)
    WvT = torch.randn(h, d_k, d_m, device='cuda').to(torch.bfloat16)
    V = torch.empty(R, h * d_k, device='cuda', dtype=torch.bfloat16)
    bias = torch.randn(h * d_k, device='cuda')
    st = torch.cuda.current_stream().cuda_stream
    # strided (shipped): A_i rows r*h+i
    f1 = lambda: capi.check(L.elattn_gpu_testing_gemm_bf16(C.data_ptr(), h * d_m, d_m, WvT.data_ptr(), d_m, d_k * d_m, V.data_ptr(), h * d_k, d_k, bias.data_ptr(), d_k, R, d_k, d_m, h, 1.0, 1, torch.cuda.current_stream().cuda_stream))
    # head-major: A_i = C[i*R:(i+1)*R]
    f2 = lambda: capi.check(L.elattn_gpu_testing_gemm_bf16(C.data_ptr(), d_m, R * d_m, WvT.data_ptr(), d_m, d_k * d_m, V.data_ptr(), h * d_k, d_k, bias.data_ptr(), d_k, R, d_k, d_m, h, 1.0, 1, torch.cuda.current_stream().cuda_stream))
    print(json.dumps({"B": B, "strided_us": round(graph_time(f1), 2), "headmajor_us": round(graph_time(f2), 2)}))
