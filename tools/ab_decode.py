"""A/B timing of the fused decode (+ split merge) between library builds on ONE box:
    python tools/ab_decode.py path/to/libA.so path/to/libB.so [--B 320 296] [--rounds 3]
Each build runs in its own process (CUDA-graph replay of back-to-back decode launches,
CUDA events); builds alternate for `rounds` rounds so clock / thermal drift hits both."""
import argparse
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs="+")
ap.add_argument("--B", type=int, nargs="+", default=[320, 296])
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--x", type=int, default=4, help="beams per input (rows = x * 16 heads)")
ap.add_argument("--child", action="store_true")
a = ap.parse_args()

if a.child:
    sys.path.insert(0, str(ROOT))
    from paper_2105_04779_b200 import capi
    capi.LIB_PATH = Path(a.libs[0]).resolve()
    import torch
    import paper_2105_04779_b200 as E
    h, d_m, d_k, x, n = 16, 1024, 64, a.x, 1024
    layer = E.ElAttentionLayer(E.AttentionParams.random(h, d_m, d_k, E.Rng(1)), E.DTYPE_BF16)
    L = capi.lib()
    res = {}
    for B in a.B:
        g = torch.Generator(device="cuda").manual_seed(B)
        H = (torch.rand((B, n, d_m), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
        Y = (torch.rand((B * x, d_m), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
        qp = layer.build_el_query(Y)
        ctx = torch.empty_like(qp)
        s = torch.cuda.Stream()
        def once():
            capi.check(L.elattn_gpu_el_attention_decode(layer.dev.handle, qp.data_ptr(), H.data_ptr(), None, B,
                                                        x * h, n, ctx.data_ptr(), s.cuda_stream))
        with torch.cuda.stream(s):
            once()
            torch.cuda.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=s):
                for _ in range(20):
                    once()
            gr.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            gr.replay()
            e1.record(s)
        torch.cuda.synchronize()
        res[B] = round(e0.elapsed_time(e1) / 20 * 1e3, 2)
        del H, qp, ctx
    print(json.dumps(res))
    sys.exit(0)

out = {lib: {B: [] for B in a.B} for lib in a.libs}
for r in range(a.rounds):
    for lib in a.libs:
        p = subprocess.run([sys.executable, __file__, lib, "--child", "--x", str(a.x), "--B", *map(str, a.B)],
                           capture_output=True,
                           text=True, cwd=ROOT)
        d = json.loads(p.stdout.strip().splitlines()[-1])
        for B in a.B:
            out[lib][B].append(d[str(B)])
for lib in a.libs:
    print(lib, {B: (min(v), v) for B, v in out[lib].items()})
