"""Steady-state per-tile cadence of the tcgen05 decode kernel (first cluster), from the
clock64 testing hook.  Prints the median cycles each role spends waiting / working per
tile, so the critical role is visible.

    python tools/trace_summary.py --B 320
"""
import argparse
import ctypes
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2105_04779_b200 import capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, nargs="+", default=[320])
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--rows", type=int, default=64)
ap.add_argument("--d_m", type=int, default=1024)
a = ap.parse_args()
L = capi.lib()
L.elattn_gpu_testing_set_decode_trace.argtypes = [ctypes.c_void_p]
L.elattn_gpu_testing_decode_bf16.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 4 + [ctypes.c_float, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
NEV, NT = 32, 64
SPANS = [  # (name, end event, start event)
    ("cadence: P(G) posted - P(G-1) posted", 13, -13),
    ("producer: wait for ring slot", 1, 0),
    ("S issuer: issue+commit of one tile", 3, 2),
    ("exchange: wait S_full", 7, 6),
    ("exchange: wait peer recv_free", 8, 7),
    ("exchange: send", 9, 8),
    ("softmax: wait S + peer scores", 11, 10),
    ("softmax: compute", 12, 11),
    ("softmax: P buffer, o_done, rescale, post", 13, 12),
    ("O issuer: wait P_full", 5, 4),
]
for B in a.B:
    d_m, rows, n = a.d_m, a.rows, a.n
    qp = (torch.randn(B * rows, d_m, device="cuda") * 0.3).to(torch.bfloat16)
    H = (torch.rand(B, n, d_m, device="cuda") * 2 - 1).to(torch.bfloat16)
    ctx = torch.empty_like(qp)
    tr = torch.zeros(2 * NEV * NT + 4096, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for i in range(3):
        L.elattn_gpu_testing_set_decode_trace(tr.data_ptr() if i == 2 else None)
        capi.check(L.elattn_gpu_testing_decode_bf16(qp.data_ptr(), H.data_ptr(), None, B, rows, n, d_m, 0.125,
                                                    ctx.data_ptr(), 1, st))
    L.elattn_gpu_testing_set_decode_trace(None)
    torch.cuda.synchronize()
    t = tr[:2 * NEV * NT].view(2, NEV, NT).cpu().numpy().astype(np.int64)
    print(f"B={B} n={n} rows={rows} d_m={d_m}  (cycles, median over steady-state tiles 4..{NT - 2})")
    for cta in range(2):
        g = np.arange(4, NT - 1)
        out = []
        for name, e1, e0 in SPANS:
            if e0 < 0:
                v = t[cta, e1, g] - t[cta, -e0, g - 1]
            else:
                v = t[cta, e1, g] - t[cta, e0, g]
            ok = (t[cta, e1, g] > 0) & (t[cta, abs(e0), g] > 0)
            v = v[ok]
            out.append(f"  cta{cta} {name:45s} med {int(np.median(v)) if len(v) else -1:6d}  p90 "
                       f"{int(np.percentile(v, 90)) if len(v) else -1:6d}")
        print("\n".join(out))
    t0 = t[0][t[0] > 0].min()
    print("  epilogue spans (li 0,1):", [(int(t[0, 14, i] - t0), int(t[0, 15, i] - t0)) for i in range(2)])
    # input transitions: events keyed by input index li (cluster 0, CTA 0), relative to the
    # softmax posting the last P of the previous input
    T = n // 32
    print("  transition li: lastP(li-1) | S_last_commit(li-1) q_empty->fill fill_done q_tma S_start(li) "
          "P0(li) o_full(li-1) epi_unit0_ld epi_loop_end epi_end(li-1) O_first(li)")
    for li in (1, 2, 3):
        if li * T + 1 > NT:
            continue
        base = t[0, 13, li * T - 1]
        if base == 0:
            continue
        r = lambda e, i: int(t[0, e, i] - base) if t[0, e, i] else None  # noqa: E731
        print(f"   li={li}: 0 | {r(3, li * T - 1)} {r(17, li)} {r(18, li)} {r(22, li)} {r(16, li)} "
              f"{r(13, li * T)} {r(19, li - 1)} {r(21, li - 1)} {r(23, li - 1)} {r(15, li - 1)} {r(20, li)}")
    # epilogue units of input li=1 (full inputs only): tmem-ld done / stage free / staged / (next)
    print("  epilogue units li=1 (rel. to o_full): m: ld_done wait_start stage_free staged stored")
    base = t[0, 19, 1]
    for m in range(4):
        i = 4 + m
        st = int(t[0, 28, i] - base) if t[0, 28, i] else None
        print(f"   m={m}: {int(t[0, 27, i] - base)} {int(t[0, 24, i] - base)} {int(t[0, 25, i] - base)} {int(t[0, 26, i] - base)} {st}")
