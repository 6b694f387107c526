"""Small-batch decoder step (BASELINE config 2 at B = 16..64): the 12-layer DecoderStep
graph timed per step with CUDA events, in two regimes:
  cold — L2 flushed (a 512 MB write) before every timed step: nothing of H survives
         from the previous step (the bench rule for inputs smaller than L2);
  warm — steps back to back: H (B * 2 MiB) may stay in L2 across steps, as it does in a
         real decode loop, where the encoder state is the same for every step.
Within one step the 12 layers re-read the same H either way.

    python tools/time_small_batch.py --B 16 32 48 64
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
ap.add_argument("--B", type=int, nargs="+", default=[16, 32, 48, 64])
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--lib", default=None, help="library build to load (A/B runs)")
a = ap.parse_args()
if a.lib:
    capi.LIB_PATH = Path(a.lib).resolve()
L, x, n, d_m = 12, 4, 1024, 1024
layers = [E.ElAttentionLayer(E.AttentionParams.random(16, d_m, 64, E.Rng(1 + l)), E.DTYPE_BF16) for l in range(L)]
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
for B in a.B:
    g = torch.Generator(device="cuda").manual_seed(B)
    H = (torch.rand((B, n, d_m), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    dec = E.DecoderStep(layers, H, B, x)
    dec.Y.copy_((torch.rand((B * x, d_m), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16))
    for _ in range(3):
        dec.run(stream=st)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.reps)]
    for e0, e1 in ev:  # cold: flush L2 between steps
        flush.fill_(1)
        e0.record(st)
        dec.run(stream=st)
        e1.record(st)
    torch.cuda.synchronize()
    cold = sorted(e0.elapsed_time(e1) for e0, e1 in ev)[a.reps // 2]
    e0, e1 = ev[0]
    e0.record(st)
    for _ in range(a.reps):
        dec.run(stream=st)
    e1.record(st)
    torch.cuda.synchronize()
    warm = e0.elapsed_time(e1) / a.reps
    print(json.dumps({"B": B, "x": x, "n": n, "layers": L, "H_MB": round(B * n * d_m * 2 / 2**20, 1),
                      "cold_step_ms": round(cold, 4), "warm_step_ms": round(warm, 4),
                      "cold_tokens_per_s": round(B * x / (cold / 1e3)), "warm_tokens_per_s": round(B * x / (warm / 1e3))}),
          flush=True)
    del dec, H
    torch.cuda.empty_cache()
