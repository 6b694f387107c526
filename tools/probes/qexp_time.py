"""Query expansion alone (graph replay, warm): fused one-launch kernel vs the two GEMMs."""
import ctypes, json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch
import paper_2105_04779_b200 as E
from paper_2105_04779_b200 import capi
L = capi.lib()
L.elattn_gpu_testing_qexp_fused.argtypes = [ctypes.c_int]
layer = E.ElAttentionLayer(E.AttentionParams.random(16, 1024, 64, E.Rng(1)), E.DTYPE_BF16)
def graph_time(fn, reps=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps): fn()
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); g.replay(); e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
for B in (4, 8, 16, 32, 64, 128):
    R = B * 4
    Y = (torch.rand((R, 1024), device="cuda") * 2 - 1).to(torch.bfloat16)
    qp = torch.empty(R * 16, 1024, device="cuda", dtype=torch.bfloat16)
    res = {"B": B}
    for mode in (1, 0):
        capi.check(L.elattn_gpu_testing_qexp_fused(mode))
        res["fused_us" if mode else "two_gemms_us"] = round(graph_time(lambda: layer.build_el_query(Y, qp)), 2)
    capi.check(L.elattn_gpu_testing_qexp_fused(-1))
    print(json.dumps(res), flush=True)
