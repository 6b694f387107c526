"""A/B timing of device beam-candidate selection between library builds on one box:
    python tools/ab_beam.py libA.so libB.so [--B 64 320] [--beam 4 12]"""
import argparse, json, subprocess, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs="+")
ap.add_argument("--B", type=int, nargs="+", default=[32, 64, 320])
ap.add_argument("--beam", type=int, nargs="+", default=[4, 12])
ap.add_argument("--child", action="store_true")
a = ap.parse_args()
if a.child:
    sys.path.insert(0, str(ROOT))
    from paper_2105_04779_b200 import capi
    capi.LIB_PATH = Path(a.libs[0]).resolve()
    import torch
    import paper_2105_04779_b200 as E
    res = {}
    for B in a.B:
        for beam in a.beam:
            lp = torch.randn(B * beam, 50265, device="cuda").log_softmax(-1)
            live = torch.randn(B * beam, device="cuda")
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                E.beam_candidates(lp, live, beam, 2 * beam, stream=s)
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    for _ in range(20):
                        E.beam_candidates(lp, live, beam, 2 * beam, stream=s)
                g.replay(); torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s); g.replay(); e1.record(s)
            torch.cuda.synchronize()
            res[f"{B}x{beam}"] = round(e0.elapsed_time(e1) / 20 * 1e3, 1)
    print(json.dumps(res)); sys.exit(0)
for lib in a.libs:
    p = subprocess.run([sys.executable, __file__, lib, "--child", "--B", *map(str, a.B), "--beam", *map(str, a.beam)],
                       capture_output=True, text=True, cwd=ROOT)
    print(lib, p.stdout.strip().splitlines()[-1] if p.stdout.strip() else p.stderr[-500:])
