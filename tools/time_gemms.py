"""CUDA-event timing of the four projection GEMM shapes of one BART layer step."""
import argparse
import ctypes
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2105_04779_b200 import capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=320)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--only", default=None, help="substring of the GEMM name to run")
ap.add_argument("--no-cublas", action="store_true")
ap.add_argument("--sweep", action="store_true", help="time every block-shape instantiation")
ap.add_argument("--tma-epilogue", action="store_true")
ap.add_argument("--kernel", type=int, default=1, help="1: tcgen05 with stream-K scratch, 2: data-parallel only")
ap.add_argument("--lib", default=None, help="library build to load (A/B runs)")
a = ap.parse_args()
if a.lib:
    capi.LIB_PATH = Path(a.lib).resolve()
L = capi.lib()
vp, i32, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
L.elattn_gpu_testing_gemm_bf16.argtypes = [vp, i64, i64, vp, i64, i64, vp, i64, i64, vp, i64,
                                           i32, i32, i32, i32, ctypes.c_float, i32, vp]
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
    "Q=Y.Wq": (Y, d_m, 0, WqT, d_m, 0, Q, h * d_k, 0, bias, 0, R, h * d_k, d_m, 1),
    "q'=Q_i.Wk_i^T": (Q, h * d_k, d_k, Wk, d_k, d_m * d_k, qp, h * d_m, d_m, None, 0, R, d_m, d_k, h),
    "V_i=C_i.Wv_i": (ctx, h * d_m, d_m, WvT, d_m, d_k * d_m, V, h * d_k, d_k, bias, d_k, R, d_k, d_m, h),
    "out=V.Wo": (V, h * d_k, 0, WoT, h * d_k, 0, out, d_m, 0, bias, 0, R, d_m, h * d_k, 1),
}


def graph_time(fn, reps):
    """device time per call: `reps` calls captured in one CUDA graph, replayed (no host gaps)"""
    gs = torch.cuda.Stream()
    gs.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(gs):
        fn()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=gs):
            for _ in range(reps):
                fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


L.elattn_gpu_testing_gemm_config.argtypes = [i32, i32, i32]
L.elattn_gpu_testing_gemm_epilogue(1 if a.tma_epilogue else -1)
CFGS = [(0, 0, 0)]
if a.sweep:
    CFGS += [(bn, mt, kbp) for bn in (64, 128, 256) for mt in (1, 2) for kbp in (1, 2)
             if not (bn == 256 and mt == 2)]
for (A, lda, sAz, Bm, ldb, sBz, C, ldc, sCz, bs, sbz, M, N, K, Z), name, cfg in [
        (v, k, c) for k, v in shapes.items() for c in CFGS]:
    if a.only and a.only not in name:
        continue
    if cfg[0] > 64 and N <= 64:
        continue
    capi.check(L.elattn_gpu_testing_gemm_config(*cfg))
    def run():
        capi.check(L.elattn_gpu_testing_gemm_bf16(A.data_ptr(), lda, sAz, Bm.data_ptr(), ldb, sBz, C.data_ptr(), ldc,
                                                  sCz, bs.data_ptr() if bs is not None else None, sbz, M, N, K, Z,
                                                  1.0, a.kernel, torch.cuda.current_stream().cuda_stream))
    run()
    torch.cuda.synchronize()
    us = graph_time(run, a.reps)
    byt = (M * K * Z + N * K * Z + M * N * Z) * 2
    print(json.dumps({"gemm": name, "cfg": cfg, "us": round(us, 2), "GBps": round(byt / us / 1e3, 1),
                      "TFLOPs": round(2 * M * N * K * Z / us / 1e6, 1)}))

capi.check(L.elattn_gpu_testing_gemm_config(0, 0, 0))
# cuBLAS (torch.matmul) on the two plain shapes, for reference
if a.no_cublas:
    raise SystemExit(0)
for name, (A, Bm) in {"cublas Q=Y.Wq": (Y, WqT), "cublas out=V.Wo": (V, WoT)}.items():
    us = graph_time(lambda: torch.matmul(A, Bm.t()), a.reps)
    print(json.dumps({"gemm": name, "us": round(us, 2)}))
qh = Q.view(R, h, d_k).transpose(0, 1)  # [h, R, d_k]
us = graph_time(lambda: torch.bmm(qh, Wk.transpose(1, 2)), a.reps)
print(json.dumps({"gemm": "cublas q' (bmm, [h][R][d_m] layout)", "us": round(us, 2)}))
ch = ctx.view(R, h, d_m).transpose(0, 1)  # [h, R, d_m]
us = graph_time(lambda: torch.bmm(ch, WvT.transpose(1, 2)), a.reps)
print(json.dumps({"gemm": "cublas V (bmm, [h][R][d_k] layout)", "us": round(us, 2)}))
