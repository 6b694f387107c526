"""Paper-style EL-attention vs multi-head-attention comparison on one B200
(the reference's MHA path is KvCache::append / attention_over_cache,
attention.hpp:118-188, with the decoder state holding per-layer caches,
model.hpp:409-416).

Decoder step of L cross-attention layers at BART-large shapes, B inputs x `beam` lanes:

  mha_expanded  fairseq-style incremental MHA: per-layer K/V caches built once per input
                (K_i = H.Wk_i + bk_i, V_i = H.Wv_i + bv_i) and replicated per beam
                ([B*x, h, n, d_k]); per step q = y.Wq + bq, SDPA over the cache, .Wo + bo.
  mha_shared    the same caches without the beam copy ([B, h, n, d_k]); the x beams of an
                input are x query rows of one SDPA call (reads each cache once per step).
  mha_ours      the same shared-cache MHA on THIS library's kernels (MhaKvCache: K/V caches
                built by the tcgen05 GEMM, mha_decode_kernel over them, tcgen05 projections),
                so EL and MHA run on the same GEMMs;
  el            this repo's EL path (DecoderStep: one CUDA graph over the L layers; H is
                the only per-input state, shared by every layer, beam and head).

The MHA baselines are library code (cuBLAS GEMMs + torch SDPA, i.e. flash / cuDNN
kernels), each step captured into a CUDA graph like the EL step.  Reported: device ms per
step (CUDA events around graph replays), tokens/s, per-input decoder-state bytes, and the
one-off cache-build time the MHA variants pay per input.

    python tools/mha_vs_el.py --B 32 320 [--layers 12] [--beam 4]
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

import paper_2105_04779_b200 as E  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, nargs="+", default=[32, 320])
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--beam", type=int, default=4)
ap.add_argument("--layers", type=int, default=12)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--skip-expanded-above-gb", type=float, default=120.0)
a = ap.parse_args()
h, d_m, d_k, x, n, L = 16, 1024, 64, a.beam, a.n, a.layers
bf = torch.bfloat16
dev = "cuda"


def graph_ms(fn, reps):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def event_ms(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


params = [E.AttentionParams.random(h, d_m, d_k, E.Rng(1 + l)) for l in range(L)]


def dense(p):
    """torch views of one layer's weights (bf16): Wq, Wk, Wv as [d_m, h*d_k], Wo [h*d_k, d_m]."""
    t = lambda w: torch.from_numpy(w).to(dev, torch.float32)  # noqa: E731
    Wq = t(p.Wq).permute(1, 0, 2).reshape(d_m, h * d_k).to(bf)
    Wk = t(p.Wk).permute(1, 0, 2).reshape(d_m, h * d_k).to(bf)
    Wv = t(p.Wv).permute(1, 0, 2).reshape(d_m, h * d_k).to(bf)
    Wo = t(p.Wo).reshape(h * d_k, d_m).to(bf)
    b = lambda v: torch.from_numpy(v).to(dev, torch.float32).reshape(-1).to(bf)  # noqa: E731
    return Wq, Wk, Wv, Wo, b(p.bq), b(p.bk), b(p.bv), b(p.bo)


W = [dense(p) for p in params]
results = []
for B in a.B:
    R = B * x
    g = torch.Generator(device=dev).manual_seed(7)
    H = (torch.rand((B, n, d_m), generator=g, device=dev) * 2 - 1).to(bf)
    Y = (torch.rand((R, d_m), generator=g, device=dev) * 2 - 1).to(bf)
    line = {"B": B, "beam": x, "n": n, "layers": L}

    # ---- EL (this repo)
    layers = [E.ElAttentionLayer(p, E.DTYPE_BF16) for p in params]
    dec = E.DecoderStep(layers, H, B, x)
    dec.Y.copy_(Y)
    for _ in range(2):
        dec.run()
    ms = event_ms(lambda: [dec.run() for _ in range(a.reps)]) / a.reps  # one graph launch per step
    el_out = dec.run().clone()
    line["el"] = {"ms_per_step": ms, "tokens_per_s": R / (ms / 1e3),
                  "state_bytes_per_input": n * d_m * 2, "cache_build_ms": 0.0}
    del dec, layers
    torch.cuda.empty_cache()

    # ---- MHA on this library's kernels: per-layer caches [h][B][n][d_k], built once
    layers = [E.ElAttentionLayer(p, E.DTYPE_BF16) for p in params]
    caches = []
    build_ms = event_ms(lambda: caches.extend(E.MhaKvCache(l, H) for l in layers))
    yb = [torch.empty(R, d_m, device=dev, dtype=bf) for _ in range(2)]

    def step_ours():
        y = Y
        for l, c in enumerate(caches):
            y = c.attend(y, out=yb[l % 2])
        return y

    ms = graph_ms(step_ours, a.reps)
    out = step_ours()
    err = ((out.float() - el_out.float()).abs().max() / el_out.float().abs().max()).item()
    line["mha_ours"] = {"ms_per_step": ms, "tokens_per_s": R / (ms / 1e3),
                        "state_bytes_per_input": L * 2 * n * h * d_k * 2, "cache_build_ms": build_ms,
                        "rel_err_vs_el": err}
    del caches, layers
    torch.cuda.empty_cache()

    # ---- MHA caches: K_i, V_i per layer (build once per input)
    def build(expand):
        Ks, Vs = [], []
        for (Wq, Wk, Wv, Wo, bq, bk, bv, bo) in W:
            K = torch.addmm(bk, H.view(B * n, d_m), Wk).view(B, n, h, d_k).transpose(1, 2)
            V = torch.addmm(bv, H.view(B * n, d_m), Wv).view(B, n, h, d_k).transpose(1, 2)
            if expand:  # beam-expanded copies, [B*x, h, n, d_k]
                K = K.unsqueeze(1).expand(B, x, h, n, d_k).reshape(B * x, h, n, d_k)
                V = V.unsqueeze(1).expand(B, x, h, n, d_k).reshape(B * x, h, n, d_k)
            else:
                K, V = K.contiguous(), V.contiguous()
            Ks.append(K)
            Vs.append(V)
        return Ks, Vs

    for mode in ("mha_shared", "mha_expanded"):
        expand = mode == "mha_expanded"
        need_gb = L * 2 * (R if expand else B) * n * h * d_k * 2 / 1e9
        if need_gb > a.skip_expanded_above_gb:
            line[mode] = {"skipped": f"cache would need {need_gb:.0f} GB"}
            continue
        built = []
        build_ms = event_ms(lambda: built.append(build(expand)))
        Ks, Vs = built[0]
        yb = [torch.empty(R, d_m, device=dev, dtype=bf) for _ in range(2)]

        def step():
            y = Y
            for l, (Wq, Wk, Wv, Wo, bq, bk, bv, bo) in enumerate(W):
                q = torch.addmm(bq, y, Wq)  # [R, h*d_k]
                if expand:
                    qh = q.view(R, h, 1, d_k)
                    o = F.scaled_dot_product_attention(qh, Ks[l], Vs[l])  # [R, h, 1, d_k]
                    o = o.reshape(R, h * d_k)
                else:
                    qh = q.view(B, x, h, d_k).transpose(1, 2)  # [B, h, x, d_k]
                    o = F.scaled_dot_product_attention(qh, Ks[l], Vs[l])  # [B, h, x, d_k]
                    o = o.transpose(1, 2).reshape(R, h * d_k)
                torch.addmm(bo, o, Wo, out=yb[l % 2])
                y = yb[l % 2]
            return y

        ms = graph_ms(step, a.reps)
        out = step()
        err = ((out.float() - el_out.float()).abs().max() / el_out.float().abs().max()).item()
        line[mode] = {"ms_per_step": ms, "tokens_per_s": R / (ms / 1e3),
                      "state_bytes_per_input": L * 2 * n * h * d_k * 2 * (x if expand else 1),
                      "cache_build_ms": build_ms, "rel_err_vs_el": err}
        del Ks, Vs, built
        torch.cuda.empty_cache()
    for mode in ("mha_ours", "mha_shared", "mha_expanded"):
        if "ms_per_step" in line.get(mode, {}):
            line[f"el_speedup_vs_{mode}"] = line[mode]["ms_per_step"] / line["el"]["ms_per_step"]
            line[f"el_state_saving_vs_{mode}"] = line[mode]["state_bytes_per_input"] / line["el"]["state_bytes_per_input"]
    print(json.dumps(line), flush=True)
    results.append(line)
