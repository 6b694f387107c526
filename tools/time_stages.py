"""Time each stage of the bf16 layer step with CUDA events (no profiler).

    python tools/time_stages.py --B 32 64 128 320
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2105_04779_b200 as E  # noqa: E402
from paper_2105_04779_b200 import capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, nargs="+", default=[32, 320])
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--x", type=int, default=4)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
h, d_m, d_k = 16, 1024, 64
p = E.AttentionParams.random(h, d_m, d_k, E.Rng(1))
layer = E.ElAttentionLayer(p, E.DTYPE_BF16)
st = torch.cuda.current_stream()
L = capi.lib()


def timeit(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us


for B in a.B:
    g = torch.Generator(device="cuda").manual_seed(0)
    H = (torch.rand(B, a.n, d_m, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    Y = (torch.rand(B * a.x, d_m, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    qp = layer.build_el_query(Y)
    ctx = torch.empty_like(qp)
    out = torch.empty_like(Y)
    dec = lambda: capi.check(L.elattn_gpu_el_attention_decode(layer.dev.handle, qp.data_ptr(), H.data_ptr(), None,  # noqa: E731
                                                              B, a.x * h, a.n, ctx.data_ptr(), st.cuda_stream))
    t_dec = timeit(dec, a.reps)
    t_q = timeit(lambda: layer.build_el_query(Y, qp), a.reps)
    t_step = timeit(lambda: layer.step(Y, H, out=out), a.reps)
    hbytes = B * a.n * d_m * 2
    print(json.dumps({"B": B, "decode_us": round(t_dec, 2), "decode_GBps": round(hbytes / t_dec / 1e3, 1),
                      "decode_frac_6545": round(hbytes / t_dec / 1e3 / 6545.6, 3),
                      "qexp_us": round(t_q, 2), "step_us": round(t_step, 2)}), flush=True)
