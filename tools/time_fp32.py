"""The fp32 (reference f32-class, <= 1e-5) layer step at BART shapes: whole step, query
expansion (Q + q' GEMMs) and the folded decode (+ V / out projections), CUDA events.

    python tools/time_fp32.py
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2105_04779_b200 as E  # noqa: E402

h, d_m, d_k, x, n = 16, 1024, 64, 4, 1024


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for B in (8, 32):
    layer = E.ElAttentionLayer(E.AttentionParams.random(h, d_m, d_k, E.Rng(1)), E.DTYPE_F32)
    H = torch.rand(B, n, d_m, device="cuda") * 2 - 1
    Y = torch.rand(B * x, d_m, device="cuda") * 2 - 1
    out = layer.step(Y, H)
    qp = layer.build_el_query(Y)
    ms_step = timed(lambda: layer.step(Y, H, out=out))
    ms_q = timed(lambda: layer.build_el_query(Y, qprime=qp))
    ms_fold = timed(lambda: layer.el_attention_folded(qp, H, x, out=out))
    print(json.dumps({"dtype": "fp32", "B": B, "layer_ms": round(ms_step, 3), "query_expansion_ms": round(ms_q, 3),
                      "folded_decode_and_projection_ms": round(ms_fold, 3),
                      "H_GBps": round(B * n * d_m * 4 / (ms_step / 1e3) / 1e9, 1)}), flush=True)

# the decoder step (12 fp32 layers over the shared H: H split once per step)
for B in (8, 32):
    layers = [E.ElAttentionLayer(E.AttentionParams.random(h, d_m, d_k, E.Rng(1 + l)), E.DTYPE_F32) for l in range(12)]
    H = torch.rand(B, n, d_m, device="cuda") * 2 - 1
    dec = E.DecoderStep(layers, H, B, x)
    dec.Y.copy_(torch.rand(B * x, d_m, device="cuda") * 2 - 1)
    ms = timed(lambda: dec.run(), reps=5)
    print(json.dumps({"dtype": "fp32", "B": B, "decoder_step_ms_12_layers": round(ms, 3),
                      "per_layer_ms": round(ms / 12, 3)}), flush=True)
    del dec, layers, H
