import sys, torch, json
sys.path.insert(0, "/root/repo")
import paper_2105_04779_b200 as E
h, d_m, d_k, x, n = 16, 1024, 64, 4, 1024
for B in (8, 32):
    layer = E.ElAttentionLayer(E.AttentionParams.random(h, d_m, d_k, E.Rng(1)), E.DTYPE_F32)
    H = torch.rand(B, n, d_m, device="cuda") * 2 - 1
    Y = torch.rand(B * x, d_m, device="cuda") * 2 - 1
    out = layer.step(Y, H); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): layer.step(Y, H, out=out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(json.dumps({"dtype": "fp32", "B": B, "layer_ms": ms, "tokens_per_s_layer": B * x / (ms / 1e3), "H_GBps": B * n * d_m * 4 / (ms / 1e3) / 1e9}))
