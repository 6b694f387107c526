"""Decode kernel alone: uniform (stream-K schedule) vs the same inputs passed with
n_per_input (strided whole-input schedule).  CUDA events, no profiler.

    python tools/time_decode_modes.py --B 32 296 320
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2105_04779_b200 as E  # noqa: E402
from paper_2105_04779_b200 import capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, nargs="+", default=[32, 296, 320])
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
h, d_m, d_k, x = 16, 1024, 64, 4
p = E.AttentionParams.random(h, d_m, d_k, E.Rng(1))
layer = E.ElAttentionLayer(p, E.DTYPE_BF16)
st = torch.cuda.current_stream()
L = capi.lib()
for B in a.B:
    g = torch.Generator(device="cuda").manual_seed(0)
    H = (torch.rand(B, a.n, d_m, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    qp = (torch.randn(B * x * h, d_m, generator=g, device="cuda") * 0.3).to(torch.bfloat16)
    ctx = torch.empty_like(qp)
    npi = torch.full((B,), a.n, dtype=torch.int32, device="cuda")
    res = {}
    for mode, ptr in (("uniform", None), ("strided", npi.data_ptr())):
        fn = lambda: capi.check(L.elattn_gpu_el_attention_decode(layer.dev.handle, qp.data_ptr(), H.data_ptr(), ptr,  # noqa: E731
                                                                 B, x * h, a.n, ctx.data_ptr(), st.cuda_stream))
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        # replay a CUDA graph of `reps` back-to-back launches: device time only, no host gaps
        gs = torch.cuda.Stream()
        gs.wait_stream(st)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(gs):
            cst = gs.cuda_stream
            fn2 = lambda: capi.check(L.elattn_gpu_el_attention_decode(layer.dev.handle, qp.data_ptr(), H.data_ptr(), ptr,  # noqa: E731
                                                                      B, x * h, a.n, ctx.data_ptr(), cst))
            fn2()  # grow this stream's scratch outside the capture
            torch.cuda.synchronize()
            with torch.cuda.graph(graph, stream=gs):
                for _ in range(a.reps):
                    fn2()
        graph.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        graph.replay()
        e1.record(st)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / a.reps * 1e3
        res[mode] = (round(us, 2), round(B * a.n * d_m * 2 / us / 1e3 / 6545.6, 3), ctx.float().sum().item())
    print(B, res, flush=True)
