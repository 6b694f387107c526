"""The GPU multi-head-attention baseline against the reference's MHA
path: K/V caches (KvCache::append, attention.hpp:134-150), attention over them
(attention_over_cache, :154-180) and the whole multi_head_attention (:96-113).

Gates as for EL: <= 1e-5 relative on the fp32 path, <= 2e-2 on bf16 with the oracle fed
the bf16-rounded inputs."""
import numpy as np
import pytest

import oracle as O
from cases import BART_CFG, make_case, make_params, rel_err, round_params

pytestmark = pytest.mark.gpu
IMPL = "reference" if O.ref_available() else "port"


def to_prod(p):
    import paper_2105_04779_b200 as E

    return E.AttentionParams(p.h, p.d_m, p.d_k, p.Wq, p.Wk, p.Wv, p.Wo, p.bq, p.bk, p.bv, p.bo,
                             p.include_key_bias, p.include_value_bias)


@pytest.mark.parametrize("h,d_m,d_k,n,g", [(1, 8, 8, 1, 1), (2, 16, 8, 7, 3), (4, 32, 8, 33, 4), (8, 64, 16, 64, 17),
                                           (4, 256, 64, 130, 16)])
@pytest.mark.parametrize("flags", [(True, True), (False, True), (True, False), (False, False)])
def test_mha_fp32_vs_reference(gpu, h, d_m, d_k, n, g, flags):
    E = gpu
    p = make_params(h, d_m, d_k, 100 + h + d_m + n)
    p.include_key_bias, p.include_value_bias = flags
    rng = O.OracleRng(7 + g)
    H = rng.uniform((n, d_m))
    q = rng.uniform((g, d_m))
    want = O.multi_head_attention(p, q, H, impl=IMPL)
    got = E.multi_head_attention(q, H, to_prod(p), E.DTYPE_F32)
    assert got.shape == want.shape
    assert rel_err(got, want) <= 1e-5


def test_mha_kv_cache_matches_reference_kvcache(gpu):
    """The device caches equal the reference's KvCache built row by row (fp32)."""
    import torch

    E = gpu
    p = make_params(4, 64, 16, 31)
    H = O.OracleRng(32).uniform((2, 9, 64))
    layer = E.ElAttentionLayer(to_prod(p), E.DTYPE_F32)
    cache = E.MhaKvCache(layer, torch.from_numpy(H).to("cuda", torch.float32))
    torch.cuda.synchronize()
    for b in range(2):
        K, V = O.kv_build(p, H[b], impl=IMPL)  # [h, t, d_k]
        assert rel_err(cache.K[:, b].double().cpu().numpy(), K) <= 1e-6
        assert rel_err(cache.V[:, b].double().cpu().numpy(), V) <= 1e-6


def test_mha_errors(gpu):
    E = gpu
    p = to_prod(make_params(2, 16, 8, 3))
    with pytest.raises(E.StateError):
        E.multi_head_attention(np.zeros((1, 16)), np.zeros((0, 16)), p)
    with pytest.raises(E.ShapeError):
        E.multi_head_attention(np.zeros((1, 12)), np.zeros((4, 16)), p)
    odd = to_prod(make_params(2, 8, 3, 4))  # d_k * 4 bytes not a multiple of 16: outside the kernel's envelope
    with pytest.raises(E.UnsupportedError):
        E.multi_head_attention(np.zeros((1, 8)), np.ones((4, 8)), odd)


def _bart_batch(B, n, x, npi=None):
    import torch

    import paper_2105_04779_b200 as E

    c = BART_CFG
    p, Y, H = make_case(c["h"], c["d_m"], c["d_k"], n, B, x)
    layer = E.ElAttentionLayer(to_prod(p), E.DTYPE_BF16)
    Hd = torch.from_numpy(H).to("cuda", torch.bfloat16)
    Yd = torch.from_numpy(Y).to("cuda", torch.bfloat16)
    nd = torch.tensor(npi, dtype=torch.int32, device="cuda") if npi is not None else None
    mha = E.MhaKvCache(layer, Hd).attend(Yd, nd)
    el = layer.step(Yd, Hd, nd)
    torch.cuda.synchronize()
    return p, Y, H, mha.double().cpu().numpy(), el.double().cpu().numpy()


def test_mha_bf16_bart_batched_vs_reference(gpu):
    """BART-large shape, 2 inputs x beam 4, n 300, bf16: the batched GPU MHA against the
    reference's multi_head_attention per input (bf16-rounded inputs), and against the EL
    path on the same inputs (EL == MHA, the paper's equivalence)."""
    from paper_2105_04779_b200.attention import round_to_dtype

    B, n, x = 2, 300, 4
    p, Y, H, mha, el = _bart_batch(B, n, x)
    pr = round_params(p, 1)
    for b in range(B):
        want = O.multi_head_attention(pr, round_to_dtype(Y[b * x:(b + 1) * x], 1), round_to_dtype(H[b], 1), impl=IMPL)
        assert rel_err(mha[b * x:(b + 1) * x], want) <= 2e-2
        # the EL path directly against the reference's MHA (north-star parity "and its MHA path")
        assert rel_err(el[b * x:(b + 1) * x], want) <= 2e-2
    assert rel_err(el, mha) <= 2e-2


def test_el_bf16_bart_full_context_vs_reference_mha(gpu):
    """The bf16 EL step at the full BART-large shape (n = 1024, beam 4) against the
    reference's own multi_head_attention (materialised per-head K/V, fp64, bf16-rounded
    inputs) — the north star's second parity target."""
    import torch

    import paper_2105_04779_b200 as E
    from paper_2105_04779_b200.attention import round_to_dtype

    c = BART_CFG
    B, n, x = 1, 1024, 4
    p, Y, H = make_case(c["h"], c["d_m"], c["d_k"], n, B, x, 41, 42)
    layer = E.ElAttentionLayer(to_prod(p), E.DTYPE_BF16)
    el = layer.step(torch.from_numpy(Y).to("cuda", torch.bfloat16), torch.from_numpy(H).to("cuda", torch.bfloat16))
    want = O.multi_head_attention(round_params(p, 1), round_to_dtype(Y, 1), round_to_dtype(H[0], 1), impl=IMPL)
    assert rel_err(el.double().cpu().numpy(), want) <= 2e-2


def test_mha_bf16_ragged_lengths(gpu):
    """n_per_input masks each input's cache: input b attends over its first n_b positions."""
    from paper_2105_04779_b200.attention import round_to_dtype

    B, n, x = 3, 64, 2
    npi = [64, 17, 1]
    p, Y, H, mha, _ = _bart_batch(B, n, x, npi)
    pr = round_params(p, 1)
    for b in range(B):
        want = O.multi_head_attention(pr, round_to_dtype(Y[b * x:(b + 1) * x], 1),
                                      round_to_dtype(H[b, :npi[b]], 1), impl=IMPL)
        assert rel_err(mha[b * x:(b + 1) * x], want) <= 2e-2
