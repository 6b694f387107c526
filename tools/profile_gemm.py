"""Run each projection GEMM of one BART layer step once (eager, no graph) so ncu can
capture them:  ncu --set full -k regex:tc_gemm python tools/profile_gemm.py --B 320"""
import argparse
import ctypes
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2105_04779_b200 import capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=320)
ap.add_argument("--cfg", type=int, nargs=3, default=[0, 0, 0])
ap.add_argument("--only", default=None)
ap.add_argument("--warm", type=int, default=2)
ap.add_argument("--kernel", type=int, default=1)
a = ap.parse_args()
L = capi.lib()
vp, i32, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
L.elattn_gpu_testing_gemm_bf16.argtypes = [vp, i64, i64, vp, i64, i64, vp, i64, i64, vp, i64,
                                           i32, i32, i32, i32, ctypes.c_float, i32, vp]
L.elattn_gpu_testing_gemm_config.argtypes = [i32, i32, i32]
h, d_m, d_k, x = 16, 1024, 64, 4
R = a.B * x
bf = torch.bfloat16
dev = "cuda"
Y = torch.randn(R, d_m, device=dev).to(bf)
Q = torch.randn(R, h * d_k, device=dev).to(bf)
qp = torch.empty(R * h, d_m, device=dev, dtype=bf)
ctx = torch.randn(R * h, d_m, device=dev).to(bf)
V = torch.empty(R, h * d_k, device=dev, dtype=bf)
out = torch.empty(R, d_m, device=dev, dtype=bf)
WqT = torch.randn(h * d_k, d_m, device=dev).to(bf)
Wk = torch.randn(h, d_m, d_k, device=dev).to(bf)
WvT = torch.randn(h, d_k, d_m, device=dev).to(bf)
WoT = torch.randn(d_m, h * d_k, device=dev).to(bf)
bias = torch.randn(max(h * d_k, d_m), device=dev)
shapes = {
    "Q": (Y, d_m, 0, WqT, d_m, 0, Q, h * d_k, 0, bias, 0, R, h * d_k, d_m, 1),
    "qp": (Q, h * d_k, d_k, Wk, d_k, d_m * d_k, qp, h * d_m, d_m, None, 0, R, d_m, d_k, h),
    "V": (ctx, h * d_m, d_m, WvT, d_m, d_k * d_m, V, h * d_k, d_k, bias, d_k, R, d_k, d_m, h),
    "O": (V, h * d_k, 0, WoT, h * d_k, 0, out, d_m, 0, bias, 0, R, d_m, h * d_k, 1),
}
capi.check(L.elattn_gpu_testing_gemm_config(*a.cfg))
for name, (A, lda, sAz, Bm, ldb, sBz, C, ldc, sCz, bs, sbz, M, N, K, Z) in shapes.items():
    if a.only and name not in a.only.split(","):
        continue
    for _ in range(a.warm + 1):
        capi.check(L.elattn_gpu_testing_gemm_bf16(A.data_ptr(), lda, sAz, Bm.data_ptr(), ldb, sBz, C.data_ptr(), ldc,
                                                  sCz, bs.data_ptr() if bs is not None else None, sbz, M, N, K, Z,
                                                  1.0, a.kernel, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
print("done")

# timeline of CTA 0 for one warm launch of each GEMM (globaltimer ns relative to kernel start)
L.elattn_gpu_testing_set_gemm_trace.argtypes = [vp]
tr = torch.zeros(64, dtype=torch.int64, device=dev)
for name, (A, lda, sAz, Bm, ldb, sBz, C, ldc, sCz, bs, sbz, M, N, K, Z) in shapes.items():
    if a.only and name not in a.only.split(","):
        continue
    tr.zero_()
    capi.check(L.elattn_gpu_testing_set_gemm_trace(tr.data_ptr()))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    capi.check(L.elattn_gpu_testing_gemm_bf16(A.data_ptr(), lda, sAz, Bm.data_ptr(), ldb, sBz, C.data_ptr(), ldc,
                                              sCz, bs.data_ptr() if bs is not None else None, sbz, M, N, K, Z,
                                              1.0, a.kernel, torch.cuda.current_stream().cuda_stream))
    e1.record()
    torch.cuda.synchronize()
    capi.check(L.elattn_gpu_testing_set_gemm_trace(None))
    t = tr.cpu().tolist()
    t0 = t[0]
    rel = lambda v: (v - t0) if v else None
    ks = [rel(v) for v in t[2:34] if v]
    print(name, "event us %.2f" % e0.elapsed_time(e1) * 1, "setup", rel(t[1]), "kstep ns", ks[:20],
          "acc", [rel(v) for v in t[34:50:2] if v], "epi_done", rel(t[50]),
          "prod_issue", [rel(v) for v in t[52:56] if v], "store_issue", [rel(v) for v in t[56:60] if v], "epi(ld,cvt,st)", [rel(v) for v in t[60:66] if v])
