"""Device beam-candidate selection (beam.cu) at BART shapes: B inputs x beam lanes x V=50265
fp32 log-probs, k = 2*beam; CUDA-graph replayed; bytes = the log-prob rows read.

    python tools/time_beam.py --B 320 --beam 4
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2105_04779_b200 as E  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, nargs="+", default=[64, 320])
ap.add_argument("--beam", type=int, nargs="+", default=[4, 12])
ap.add_argument("--V", type=int, default=50265)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
for B in a.B:
    for beam in a.beam:
        lp = torch.randn(B * beam, a.V, device="cuda").log_softmax(-1)
        live = torch.randn(B * beam, device="cuda")
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            E.beam_candidates(lp, live, beam, 2 * beam, stream=s)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                E.beam_candidates(lp, live, beam, 2 * beam, stream=s)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(a.reps):
                g.replay()
            e1.record(s)
            torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / a.reps * 1e3
        tk = torch.topk((lp + live[:, None]).view(B, -1), 2 * beam, dim=1)  # torch reference timing
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.reps):
            torch.topk((lp + live[:, None]).view(B, -1), 2 * beam, dim=1)
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"B": B, "beam": beam, "V": a.V, "k": 2 * beam, "us": us,
                          "GBps": lp.numel() * 4 / (us * 1e-6) / 1e9,
                          "torch_add_topk_us": e0.elapsed_time(e1) / a.reps * 1e3}), flush=True)
