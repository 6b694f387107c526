"""Per-tile clock64 timeline of the first cluster of the tcgen05 decode kernel."""
import argparse
import ctypes
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2105_04779_b200 import capi  # noqa: E402

EV = ["prod_wait_empty", "prod_got_empty", "S_start", "S_committed", "O_wait_pfull", "O_got_pfull",
      "X_start", "X_got_sfull", "X_got_recvfree", "X_sent", "B_start", "B_got_recv", "B_computed",
      "B_pfull_arrived", "epi_start", "epi_end", "S_u0_wait", "S_u0_ready", "S_uL_ready", "S_issued"]
ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=32)
ap.add_argument("--n", type=int, default=1024)
a = ap.parse_args()
L = capi.lib()
L.elattn_gpu_testing_set_decode_trace.argtypes = [ctypes.c_void_p]
L.elattn_gpu_testing_decode_bf16.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 4 + [ctypes.c_float, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
B, rows, n, d_m = a.B, 64, a.n, 1024
qp = (torch.randn(B * rows, d_m, device="cuda") * 0.3).to(torch.bfloat16)
H = (torch.rand(B, n, d_m, device="cuda") * 2 - 1).to(torch.bfloat16)
ctx = torch.empty_like(qp)
tr = torch.zeros(2 * 32 * 64 + 4096, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for i in range(3):
    L.elattn_gpu_testing_set_decode_trace(tr.data_ptr() if i == 2 else None)
    capi.check(L.elattn_gpu_testing_decode_bf16(qp.data_ptr(), H.data_ptr(), None, B, rows, n, d_m, 0.125,
                                                ctx.data_ptr(), 1, st))
L.elattn_gpu_testing_set_decode_trace(None)
torch.cuda.synchronize()
t = tr.view(2, 32, 64).cpu().numpy()
t0 = t[0][t[0] > 0].min()
for cta in range(1):
    print("cta", cta)
    print("tile " + " ".join(f"{e[:9]:>9}" for e in EV))
    print("epilogue start/end", t[cta, 14, 0] - t0, t[cta, 15, 0] - t0)
    print("tile   S_start  u0_wait u0_ready uL_ready  S_issued S_commit  prod_got")
    for j in range(0, 33):
        print(f"{j:4d} " + " ".join(f"{(t[cta, e, j] - t0) if t[cta, e, j] else -1:8d}" for e in (2, 16, 17, 18, 19, 3, 1)))
    for j in range(0, 33):
        vals = [t[cta, e, j] for e in range(len(EV))]
        print(f"{j:4d} " + " ".join(f"{(v - t0) if v else -1:9d}" for v in vals))
