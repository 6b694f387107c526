"""BASELINE config 4: decoder-only (GPT-2 medium shapes: d_m 1024, 16 heads, 24 layers)
EL self-attention over per-lane hidden-state caches, beam 4, as the history grows.

Per decoder step and layer: append the lane's input to its cache (device), EL attention of
the lane over its own history (x = 1, ragged lengths), and — once per step — the beam
reorder (gather_lanes on every layer's cache).  Device time per step from CUDA-graph
replays (the graph resets the lengths first, so every replay sees the same n).

    python tools/selfattn_bench.py --B 64 --n 128 512 1024

Then the reference's own decoder-only form, mixed self-attention (EL over the prefix shared
by an input's beams + a per-lane K/V cache of the generated tokens, one joint softmax):
per step and layer KvCache::append + mixed attention, for a few (prefix, generated) sizes.
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2105_04779_b200 as E  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=64)
ap.add_argument("--beam", type=int, default=4)
ap.add_argument("--layers", type=int, default=24)
ap.add_argument("--n", type=int, nargs="+", default=[128, 512, 1024])
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
h, d_m, d_k = 16, 1024, 64
lanes, L, n_max = a.B * a.beam, a.layers, max(a.n) + 1
layers = [E.ElAttentionLayer(E.AttentionParams.random(h, d_m, d_k, E.Rng(100 + l)), E.DTYPE_BF16) for l in range(L)]
cache = E.HiddenStateCache(L, lanes, n_max, d_m, E.DTYPE_BF16)
g = torch.Generator(device="cuda").manual_seed(3)
cache.cache.copy_((torch.rand(cache.cache.shape, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16))
Y = (torch.rand((lanes, d_m), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
outs = [torch.empty_like(Y) for _ in range(2)]
parent = torch.arange(lanes, device="cuda", dtype=torch.int32).view(a.B, a.beam).flip(1).reshape(-1)
# a beam-search-like reorder: each lane continues a random beam of its own input (parents
# repeat, some beams die) — copy-on-fork copies one history per extra child
gp = torch.Generator().manual_seed(7)
parent_beam = (torch.arange(a.B).view(a.B, 1) * a.beam + torch.randint(0, a.beam, (a.B, a.beam), generator=gp))
parent_beam = parent_beam.reshape(-1).to(torch.int32).cuda()


def timed(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            fn()
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.reps


for n in a.n:
    base = torch.full((L, lanes), n - 1, dtype=torch.int32, device="cuda")

    def step_attn():
        cache.lengths.copy_(base)
        y = Y
        for l in range(L):
            cache.append(l, y)
            y = cache.attend(layers[l], l, y, out=outs[l % 2])

    def step_gather():
        cache.gather(parent, rows_hint=n)

    def step_gather_beam():
        cache.gather(parent_beam, rows_hint=n)

    ms_attn = timed(step_attn)
    cache.lengths.copy_(base + 1)
    ms_gather = timed(step_gather)
    ms_gather_beam = timed(step_gather_beam)
    byt = L * lanes * n * d_m * 2  # every lane's history read once per layer
    print(json.dumps({"config": "GPT-2 medium decoder-only, hidden-state-only cache", "B": a.B, "beam": a.beam,
                      "lanes": lanes, "layers": L, "n": n, "attn_ms_per_step": ms_attn,
                      "tokens_per_s": lanes / (ms_attn / 1e3), "history_GBps": byt / (ms_attn / 1e3) / 1e9,
                      "gather_ms_per_step": ms_gather, "gather_parent": "permutation (beams reversed)",
                      "gather_beam_ms_per_step": ms_gather_beam,
                      "gather_beam_copies": int(a.beam * a.B - sum(len(set(r)) for r in parent_beam.view(a.B, a.beam).tolist())),
                      "cache_GB": cache.cache.numel() * 2 / 1e9}), flush=True)

# ---- the reference's decoder-only EL form: mixed self-attention (EL over the prefix shared
# by an input's beams + per-lane K/V cache of generated tokens, joint softmax;
# attention.hpp:309-365), per step: KvCache::append + mixed attention on every layer
for n_in, t_out in ((512, 64), (512, 256), (1024, 128)):
    P = (torch.rand((a.B, n_in, d_m), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    caches = [E.KvCache(layers[l], lanes, t_out + 1) for l in range(L)]
    for c in caches:  # pre-fill t_out - 1 generated rows
        c.K.copy_((torch.rand(c.K.shape, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16))
        c.V.copy_((torch.rand(c.V.shape, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16))

    def step_mixed():
        y = Y
        for l in range(L):
            caches[l].t = t_out - 1
            caches[l].append(y)
            y = E.mixed_self_attention_batched(layers[l], y, P, caches[l], a.beam, out=outs[l % 2])

    ms = timed(step_mixed)
    byt = L * (a.B * n_in * d_m * 2 + 2 * lanes * t_out * d_m * 2)  # prefix once per input + K/V of every lane
    print(json.dumps({"config": "GPT-2 medium decoder-only, mixed self-attention (EL prefix + K/V generated)",
                      "B": a.B, "beam": a.beam, "lanes": lanes, "layers": L, "prefix_n": n_in, "generated_t": t_out,
                      "ms_per_step": ms, "tokens_per_s": lanes / (ms / 1e3),
                      "state_GBps": byt / (ms / 1e3) / 1e9}), flush=True)
