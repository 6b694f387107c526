"""Ragged batches: the fused decode alone (CUDA-graph replay, CUDA events) for per-input
context lengths n_b drawn from [288, 1024] (mean 640) against a uniform batch with the same
total number of H tiles (n_b = 640 for every input), under the automatic schedule (ragged
stream-K on request, longest-first whole inputs by default) and under whole-input
striding (the previous ragged schedule).

    python tools/time_ragged.py --B 128 320
"""
import argparse
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2105_04779_b200 as E  # noqa: E402
from paper_2105_04779_b200 import capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, nargs="+", default=[64, 128, 320])
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
h, d_m, d_k, x, n = 16, 1024, 64, 4, 1024
layer = E.ElAttentionLayer(E.AttentionParams.random(h, d_m, d_k, E.Rng(1)), E.DTYPE_BF16)
L = capi.lib()
L.elattn_gpu_testing_decode_sched.argtypes = [ctypes.c_int]


def time_decode(qp, H, npi, B, ctx, n_arg=n):
    s = torch.cuda.Stream()
    def once():
        capi.check(L.elattn_gpu_el_attention_decode(layer.dev.handle, qp.data_ptr(), H.data_ptr(),
                                                    npi.data_ptr() if npi is not None else None, B, x * h, n_arg,
                                                    ctx.data_ptr(), s.cuda_stream))
    with torch.cuda.stream(s):
        once()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(a.reps):
                once()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.reps * 1e3


for B in a.B:
    rng = np.random.default_rng(B)
    lens = rng.integers(288, 1025, B)
    lens = np.clip(np.round(lens * (640 * B / lens.sum())), 1, n).astype(np.int32)  # mean 640
    g = torch.Generator(device="cuda").manual_seed(B)
    H = (torch.rand((B, n, d_m), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    Y = (torch.rand((B * x, d_m), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    qp = layer.build_el_query(Y)
    ctx = torch.empty_like(qp)
    rag = torch.from_numpy(lens).cuda()
    uni = torch.full((B,), 640, dtype=torch.int32, device="cuda")
    res = {"B": B, "tiles_ragged": int(((lens + 31) // 32).sum()), "tiles_uniform": B * 20}
    for mode, name in ((0, "auto"), (2, "whole"), (1, "streamk")):
        capi.check(L.elattn_gpu_testing_decode_sched(mode))
        res[f"uniform640_{name}_us"] = round(time_decode(qp, H, uni, B, ctx), 2)
        res[f"ragged_{name}_us"] = round(time_decode(qp, H, rag, B, ctx), 2)
    capi.check(L.elattn_gpu_testing_decode_sched(0))
    res["ratio_auto"] = round(res["ragged_auto_us"] / res["uniform640_auto_us"], 3)
    res["ratio_whole"] = round(res["ragged_whole_us"] / res["uniform640_whole_us"], 3)
    # the same total tiles without n_per_input (uniform n = 640): the schedule a uniform batch gets
    res["uniform640_nonpi_us"] = round(time_decode(qp[: B * x * h].contiguous(), H[:, :640].contiguous(), None, B,
                                                   ctx, n_arg=640), 2)
    res["ratio_vs_uniform_nonpi"] = round(res["ragged_auto_us"] / res["uniform640_nonpi_us"], 3)
    print(json.dumps(res), flush=True)
