"""In-graph timeline of one 12-layer decoder step, per kernel launch, from a measurement
build of the library (per-CTA %globaltimer records, csrc/timeline.cuh):

    cd paper_2105_04779_b200/csrc && make BUILD=build_tl LIB=build_tl/libtl.so EXTRA=-DELA_TIMELINE
    python tools/step_timeline.py --B 32 320

Per launch (in start order): CTAs, first entry, median / last PDL-wait release, first /
median / last exit — relative to the step's first entry, in microseconds.  `gap` is the
time from the previous launch's last exit to this launch's first PDL-wait release (negative:
the data phase could not start before the predecessor completed, so this is the
dependency bubble)."""
import argparse
import ctypes
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2105_04779_b200 import capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, nargs="+", default=[32])
ap.add_argument("--x", type=int, default=4)
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--layers", type=int, default=12)
ap.add_argument("--lib", default=str(ROOT / "paper_2105_04779_b200/csrc/build_tl/libtl.so"))
ap.add_argument("--show", type=int, default=12, help="launches to print (the rest summarised)")
ap.add_argument("--json", default=None)
ap.add_argument("--dump", type=int, nargs="*", default=[], help="launch indices to print per CTA")
a = ap.parse_args()
capi.LIB_PATH = Path(a.lib).resolve()
import paper_2105_04779_b200 as E  # noqa: E402

L = capi.lib()
L.elattn_gpu_testing_timeline.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint]
KIND = {1: "gemm", 2: "splitk", 3: "qexp", 4: "decode", 5: "merge"}
CAP = 1 << 16
layers = [E.ElAttentionLayer(E.AttentionParams.random(16, 1024, 64, E.Rng(1 + l)), E.DTYPE_BF16)
          for l in range(a.layers)]
st = torch.cuda.current_stream()
out = []
for B in a.B:
    g = torch.Generator(device="cuda").manual_seed(B)
    H = (torch.rand((B, a.n, 1024), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    dec = E.DecoderStep(layers, H, B, a.x)
    dec.Y.copy_((torch.rand((B * a.x, 1024), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16))
    rec = torch.zeros(CAP * 8, dtype=torch.int64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    for _ in range(3):
        dec.run(stream=st)
    torch.cuda.synchronize()
    capi.check(L.elattn_gpu_testing_timeline(rec.data_ptr(), cnt.data_ptr(), CAP))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    dec.run(stream=st)
    e1.record(st)
    torch.cuda.synchronize()
    capi.check(L.elattn_gpu_testing_timeline(None, None, 0))
    n = min(int(cnt.item()), CAP)
    r = rec[: n * 8].view(n, 8).cpu().numpy()
    entry, wait, exit_ = r[:, 0].astype(np.int64), r[:, 1].astype(np.int64), r[:, 2].astype(np.int64)
    marks = r[:, 3:7].astype(np.int64)
    kind = (r[:, 7] & 0xFFFFFFFF).astype(np.int64)
    block = (r[:, 7] >> 32).astype(np.int64)
    t0 = entry.min()
    order = np.argsort(entry, kind="stable")
    launches = []  # per kind: the current launch (block ids seen)
    cur = {}
    for i in order:
        k = int(kind[i])
        c = cur.get(k)
        if c is None or int(block[i]) in c["blocks"]:
            c = {"kind": k, "blocks": set(), "idx": []}
            cur[k] = c
            launches.append(c)
        c["blocks"].add(int(block[i]))
        c["idx"].append(i)
    rows = []
    prev_end = None
    for c in launches:
        ii = np.array(c["idx"])
        en, wa, ex = (entry[ii] - t0) / 1e3, (wait[ii] - t0) / 1e3, (exit_[ii] - t0) / 1e3
        row = {"kind": KIND.get(c["kind"], c["kind"]), "ctas": len(ii), "entry0": en.min(), "entry1": en.max(),
               "wait_med": float(np.median(wa)), "wait1": wa.max(), "exit0": ex.min(), "exit_med": float(np.median(ex)),
               "exit1": ex.max(), "gap": None if prev_end is None else wa.min() - prev_end,
               "busy_med": float(np.median(ex - wa)),
               # kernel phase ends (timeline.cuh ELA_TL_MARK), median over CTAs, from the wait release
               "marks": [None if not (marks[ii, k] > 0).any() else
                         float(np.median((marks[ii, k][marks[ii, k] > 0] - wait[ii][marks[ii, k] > 0]) / 1e3))
                         for k in range(4)]}
        prev_end = ex.max()
        if len(rows) in a.dump:
            print(f"  launch {len(rows)} ({row['kind']}) per CTA (block: entry wait marks... exit, us):")
            for i in ii[np.argsort(block[ii])]:
                mk = " ".join("-" if marks[i, k] == 0 else f"{(marks[i, k] - t0) / 1e3:7.2f}" for k in range(4))
                print(f"    {block[i]:4d}: {(entry[i] - t0) / 1e3:7.2f} {(wait[i] - t0) / 1e3:7.2f} {mk} {(exit_[i] - t0) / 1e3:7.2f}")
        rows.append(row)
    step_us = e0.elapsed_time(e1) * 1e3
    print(f"B={B}: step {step_us:.1f} us (event), {len(rows)} launches, last exit {rows[-1]['exit1']:.1f} us")
    print("   kind    ctas  entry0  entry1  wait_med  exit0  exit_med  exit1   gap  busy_med  marks(from wait)")
    for row in rows[: a.show]:
        print(f"  {row['kind']:7s} {row['ctas']:5d} {row['entry0']:7.2f} {row['entry1']:7.2f} {row['wait_med']:8.2f} "
              f"{row['exit0']:6.2f} {row['exit_med']:8.2f} {row['exit1']:6.2f} "
              f"{'' if row['gap'] is None else format(row['gap'], '6.2f'):>6s} {row['busy_med']:8.2f}  "
              + " ".join("-" if m is None else f"{m:.2f}" for m in row["marks"]))
    # per kind: duration from the predecessor's end to this launch's end (its share of the step)
    share = {}
    for i, row in enumerate(rows):
        d = row["exit1"] - (rows[i - 1]["exit1"] if i else 0.0)
        share.setdefault(row["kind"], []).append(d)
    print("  share of the step by kind (sum of end-to-end increments, us):",
          {k: round(sum(v), 1) for k, v in share.items()}, " per launch:",
          {k: round(float(np.median(v)), 2) for k, v in share.items()})
    out.append({"B": B, "step_us": step_us, "launches": rows})
    del dec, H
    torch.cuda.empty_cache()
if a.json:
    Path(a.json).write_text("\n".join(json.dumps(o, default=float) for o in out) + "\n")
