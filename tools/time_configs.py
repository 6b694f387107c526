"""BASELINE.json configs 2, 3 and 5 on one B200: the whole decoder step through the public
batched API (DecoderStep: L layers over the shared H, one CUDA-graph launch), replayed
between CUDA events — device time, no host gaps.

    python tools/time_configs.py
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2105_04779_b200 as E  # noqa: E402
from paper_2105_04779_b200 import capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--lib", default=None, help="library build to load (A/B runs)")
ap.add_argument("--only", default=None, help="substring of the config name")
ap.add_argument("--B", type=int, nargs="*", default=None, help="batch sizes (default: per config)")
a = ap.parse_args()
if a.lib:
    capi.LIB_PATH = Path(a.lib).resolve()

CONFIGS = [  # (name, d_m, h, x, n, B list)
    ("2 BART-large beam 4", 1024, 16, 4, 1024, [32, 64, 128, 320]),
    ("3 Transformer-big greedy", 1024, 16, 1, 512, [64, 512, 4096]),
    ("5 diverse beam 12", 1024, 16, 12, 1024, [32, 160, 320]),
]
L, REPS, HBM = 12, 10, 6545.6e9
layers = [E.ElAttentionLayer(E.AttentionParams.random(16, 1024, 64, E.Rng(1 + l)), E.DTYPE_BF16) for l in range(L)]
for name, d_m, h, x, n, Bs in CONFIGS:
    if a.only and a.only not in name:
        continue
    for B in (a.B or Bs):
        g = torch.Generator(device="cuda").manual_seed(B)
        H = (torch.rand((B, n, d_m), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
        dec = E.DecoderStep(layers, H, B, x)
        dec.Y.copy_((torch.rand((B * x, d_m), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16))
        st = torch.cuda.current_stream()
        for _ in range(3):
            dec.run(stream=st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(REPS):
            dec.run(stream=st)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / REPS
        layer_us = ms * 1e3 / L
        h_bytes = B * n * d_m * 2
        print(json.dumps({"config": name, "B": B, "x": x, "n": n, "step_ms": round(ms, 3),
                          "layer_us": round(layer_us, 1), "tokens_per_s": round(B * x / (ms / 1e3)),
                          "H_frac_of_hbm_per_layer": round(h_bytes / (layer_us * 1e-6) / HBM, 3)}), flush=True)
        del dec, H
        torch.cuda.empty_cache()
