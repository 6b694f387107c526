"""One 12-layer DecoderStep (graph) at batch B, for ncu launch lists:
    ncu --metrics gpu__time_duration.sum --clock-control none --graph-profiling node \
        python tools/profile_step.py --B 32"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2105_04779_b200 as E  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=32)
ap.add_argument("--x", type=int, default=4)
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--steps", type=int, default=2)
a = ap.parse_args()
layers = [E.ElAttentionLayer(E.AttentionParams.random(16, 1024, 64, E.Rng(1 + l)), E.DTYPE_BF16) for l in range(12)]
g = torch.Generator(device="cuda").manual_seed(a.B)
H = (torch.rand((a.B, a.n, 1024), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
dec = E.DecoderStep(layers, H, a.B, a.x)
for _ in range(a.steps):
    dec.run()
torch.cuda.synchronize()
print("ok")
