"""Launch the fused decode kernel alone at the bench shape (for ncu captures)."""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2105_04779_b200 as E  # noqa: E402
from paper_2105_04779_b200 import capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=320)
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--x", type=int, default=4)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--step", action="store_true", help="run the whole layer step instead")
a = ap.parse_args()
h, d_m, d_k = 16, 1024, 64
p = E.AttentionParams.random(h, d_m, d_k, E.Rng(1))
layer = E.ElAttentionLayer(p, E.DTYPE_BF16)
g = torch.Generator(device="cuda").manual_seed(0)
H = (torch.rand(a.B, a.n, d_m, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
Y = (torch.rand(a.B * a.x, d_m, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
qp = layer.build_el_query(Y)
ctx = torch.empty_like(qp)
st = torch.cuda.current_stream()
for _ in range(a.reps):
    if a.step:
        layer.step(Y, H)
    else:
        capi.check(capi.lib().elattn_gpu_el_attention_decode(layer.dev.handle, qp.data_ptr(), H.data_ptr(), None,
                                                             a.B, a.x * h, a.n, ctx.data_ptr(), st.cuda_stream))
torch.cuda.synchronize()
print("ok")
