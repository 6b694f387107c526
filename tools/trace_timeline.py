"""Whole-kernel timeline of the tcgen05 decode's first cluster (clock64 testing hook):
kernel entry, setup done, first H load issued / first P posted, each segment's tiles and
epilogue span, exit — in cycles from entry, per CTA of the cluster.  Shows where a small
batch's decode time goes outside the steady tile loop.

    python tools/trace_timeline.py --B 32 320
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
ap.add_argument("--B", type=int, nargs="+", default=[32])
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--rows", type=int, default=64)
ap.add_argument("--d_m", type=int, default=1024)
ap.add_argument("--lib", default=None)
ap.add_argument("--cold", action="store_true")
ap.add_argument("--traced", type=int, default=3)
a = ap.parse_args()
if a.lib:
    capi.LIB_PATH = Path(a.lib).resolve()
L = capi.lib()
L.elattn_gpu_testing_set_decode_trace.argtypes = [ctypes.c_void_p]
L.elattn_gpu_testing_decode_bf16.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 4 + [ctypes.c_float, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
NEV, NT = 32, 64
for B in a.B:
    d_m, rows, n = a.d_m, a.rows, a.n
    qp = (torch.randn(B * rows, d_m, device="cuda") * 0.3).to(torch.bfloat16)
    H = (torch.rand(B, n, d_m, device="cuda") * 2 - 1).to(torch.bfloat16)
    ctx = torch.empty_like(qp)
    tr = torch.zeros(2 * NEV * NT + 4096, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda") if a.cold else None
    for i in range(2 + a.traced):  # the traced (instrumented) kernel runs `traced` times, the last one counts:
        # its code is then in L2 as the production kernel's is in a decoder step
        if flush is not None and i == 1 + a.traced:
            flush.fill_(1)  # cold: H not in L2 (the decoder step's case above 48 MB of H)
        L.elattn_gpu_testing_set_decode_trace(tr.data_ptr() if i >= 2 else None)
        capi.check(L.elattn_gpu_testing_decode_bf16(qp.data_ptr(), H.data_ptr(), None, B, rows, n, d_m, 0.125,
                                                    ctx.data_ptr(), 1, st))
    L.elattn_gpu_testing_set_decode_trace(None)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        capi.check(L.elattn_gpu_testing_decode_bf16(qp.data_ptr(), H.data_ptr(), None, B, rows, n, d_m, 0.125,
                                                    ctx.data_ptr(), 1, st))
    e1.record()
    torch.cuda.synchronize()
    t = tr[:2 * NEV * NT].view(2, NEV, NT).cpu().numpy().astype(np.int64)
    print(f"B={B}: eager launch (incl. merge) {e0.elapsed_time(e1) / 10 * 1e3:.1f} us")
    for cta in range(2):
        c = t[cta]
        t0 = c[29, 0]
        rel = lambda v: int(v - t0) if v else None  # noqa: E731
        posts = [rel(v) for v in c[13] if v]
        loads = [rel(v) for v in c[1] if v]
        print(f"  cta{cta}: setup {rel(c[30, 0])}  first load {loads[:1]}  P posts {len(posts)}: first {posts[:3]} "
              f"last {posts[-1:]}  exit {rel(c[31, 0])}")
        ev = lambda e, i: rel(c[e, i])  # noqa: E731
        print(f"    first input: q' TMA {ev(22, 0)}  fill {ev(17, 0)}..{ev(18, 0)}  S issuer sees q' {ev(16, 0)}")
        for G in (0, 1, 2):
            print(f"    tile {G}: load wait/issue {ev(0, G)}/{ev(1, G)}  S {ev(2, G)}..{ev(3, G)}  "
                  f"xchg sfull {ev(7, G)} recvfree {ev(8, G)} sent {ev(9, G)}  softmax S+peer {ev(11, G)} "
                  f"done {ev(12, G)} P {ev(13, G)}  O wait/go {ev(4, G)}/{ev(5, G)}")
        for li in range(8):
            if c[14, li]:
                print(f"    segment {li}: epilogue {rel(c[14, li])} .. {rel(c[15, li])}")
        if len(posts) > 4:
            d = np.diff(np.array([v for v in posts]))
            print(f"    P cadence median {int(np.median(d))} cycles, max {int(d.max())}")
    # every CTA: %globaltimer entry / exit (ns)
    gt = tr[4096:].view(-1, 2).cpu().numpy().astype(np.int64)
    gt = gt[gt[:, 0] > 0]
    g0 = gt[:, 0].min()
    ent, ex = (gt[:, 0] - g0) / 1e3, (gt[:, 1] - g0) / 1e3
    body = ex - ent
    print(f"  {len(gt)} CTAs: entry {ent.min():.2f}..{ent.max():.2f} us, exit {ex.min():.2f}..{ex.max():.2f} us, "
          f"body median {np.median(body):.2f} max {body.max():.2f} us")
