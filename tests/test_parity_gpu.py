"""Parity of the CUDA path (through the C ABI) against the oracle / reference goldens.

Gates (BASELINE.json north_star): relative error max|gpu-ref|/max|ref| <= 1e-5 on
the fp32 path, <= 2e-2 on the bf16 path; row bookkeeping exact.  For bf16 the
oracle receives the bf16-rounded inputs and weights, so the measured error is
kernel arithmetic only; the unrounded reference is checked too.
"""
import json
from pathlib import Path

import numpy as np
import pytest

import oracle as O
from cases import BART_CFG, BEAM12_CFG, ORACLE_CFG, TBIG_GREEDY_CFG, make_case, rel_err, round_params

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"
TOL = {0: 1e-5, 1: 2e-2}


def to_prod(p):
    import paper_2105_04779_b200 as E

    return E.AttentionParams(p.h, p.d_m, p.d_k, p.Wq, p.Wk, p.Wv, p.Wo, p.bq, p.bk, p.bv, p.bo,
                             p.include_key_bias, p.include_value_bias)


def run_step(E, p, Y, H, x, dtype, npi=None):
    import torch

    layer = E.ElAttentionLayer(to_prod(p), dtype)
    td = torch.bfloat16 if dtype == E.DTYPE_BF16 else torch.float32
    Yd = torch.from_numpy(Y).to("cuda", td)
    Hd = torch.from_numpy(H).to("cuda", td)
    nd = torch.from_numpy(np.asarray(npi, np.int32)).cuda() if npi is not None else None
    out = layer.step(Yd, Hd, nd)
    torch.cuda.synchronize()
    return out.double().cpu().numpy(), layer


def oracle_inputs(p, Y, H, dtype):
    from paper_2105_04779_b200.attention import round_to_dtype

    return round_params(p, dtype), round_to_dtype(Y, dtype), round_to_dtype(H, dtype)


# ---------------------------------------------------------------- fp32 path
def test_fp32_oracle_config_vs_reference_golden(gpu):
    E = gpu
    g = np.load(GOLD / "step_oracle_cfg.npz")
    c = ORACLE_CFG
    p, Y, H = make_case(c["h"], c["d_m"], c["d_k"], c["n"], c["B"], c["x"])
    out, _ = run_step(E, p, Y, H, c["x"], E.DTYPE_F32)
    assert out.shape == g["out"].shape
    assert rel_err(out, g["out"]) <= TOL[0]


def test_fp32_sweep_el_and_mha_golden(gpu):
    """test_attention.cpp:230-247 shapes (d_k = 3, n = 1 included) through el_attention."""
    E = gpu
    g = np.load(GOLD / "sweep_el_mha.npz")
    off = 0
    for seed, h, d_m, d_k, n in g["cases"]:
        rng = O.OracleRng(int(seed))
        p = O.params_random(int(h), int(d_m), int(d_k), rng)
        q = rng.uniform((1, int(d_m)))
        Hh = rng.uniform((int(n), int(d_m)))
        out = E.el_attention(q, Hh, to_prod(p), E.DTYPE_F32).ravel()
        for key in ("el", "mha"):
            assert rel_err(out, g[key][off:off + d_m]) <= TOL[0], (seed, h, d_m, d_k, n, key)
        off += int(d_m)


def test_fp32_build_el_query_and_folded_golden(gpu):
    E = gpu
    g = np.load(GOLD / "build_el_query.npz")
    p = O.params_random(3, 12, 4, O.OracleRng(53))
    eq = E.build_el_query(g["q"], to_prod(p), E.DTYPE_F32)
    assert rel_err(eq.elq, g["elq"]) <= TOL[0]
    assert np.max(np.abs(eq.s - g["s"])) <= 1e-5 * max(1.0, np.max(np.abs(g["s"])))
    f = np.load(GOLD / "folded_g4.npz")
    p = O.params_random(4, 16, 4, O.OracleRng(71))
    # the reference's own EL-Q rows fed to the GPU el_attention_folded
    out = E.el_attention_folded(f["elq"], f["H"], f["s"], to_prod(p), E.DTYPE_F32)
    assert rel_err(out, f["folded"]) <= TOL[0]
    # and the GPU query expansion end to end
    qs = [E.build_el_query(f["q"][b:b + 1], to_prod(p), E.DTYPE_F32) for b in range(4)]
    Q, S = E.fold_el_queries(qs, 4, 16)
    assert rel_err(Q, f["elq"]) <= TOL[0]
    assert rel_err(E.el_attention_folded(Q, f["H"], S, to_prod(p), E.DTYPE_F32), f["singles"]) <= TOL[0]


def test_fp32_known_answers(gpu):
    E = gpu
    d_m = 4
    I = np.eye(d_m)[None]
    z = np.zeros((1, d_m))
    p = E.AttentionParams(1, d_m, d_m, I, I, I, I, z, z, z, np.zeros(d_m))
    H = O.OracleRng(61).uniform((5, d_m))
    out = E.el_attention(np.zeros((1, d_m)), H, p, E.DTYPE_F32)  # row mean of H
    assert np.max(np.abs(out[0] - H.mean(axis=0))) <= 1e-6
    H1 = O.OracleRng(7).uniform((1, d_m))  # n = 1 -> the single row
    assert np.max(np.abs(E.el_attention(O.OracleRng(5).uniform((1, d_m)), H1, p, E.DTYPE_F32) - H1)) <= 1e-6


def test_errors_are_reference_types(gpu):
    E = gpu
    p = to_prod(O.params_random(4, 16, 4, O.OracleRng(71)))
    H = O.OracleRng(72).uniform((9, 16))
    with pytest.raises(E.ShapeError):
        E.el_attention_folded(O.OracleRng(90).uniform((6, 16)), H, np.zeros(6), p)
    with pytest.raises(E.StateError):
        E.el_attention(np.zeros((1, 16)), np.zeros((0, 16)), p)
    with pytest.raises(E.ShapeError):
        E.el_attention(np.zeros((1, 12)), H, p)


# ---------------------------------------------------------------- bf16 path
BEAM5_CFG = dict(BART_CFG, x=5)    # 80 query rows per input: a partial second 64-row virtual input
BEAM10_CFG = dict(BART_CFG, x=10)  # 160 rows


@pytest.mark.parametrize("cfg,B", [(BART_CFG, 2), (ORACLE_CFG, 2), (TBIG_GREEDY_CFG, 3), (BEAM12_CFG, 1),
                                   (BEAM5_CFG, 3), (BEAM10_CFG, 2)])
def test_bf16_step_vs_oracle(gpu, cfg, B):
    E = gpu
    p, Y, H = make_case(cfg["h"], cfg["d_m"], cfg["d_k"], cfg["n"], B, cfg["x"])
    out, layer = run_step(E, p, Y, H, cfg["x"], E.DTYPE_BF16)
    pr, Yr, Hr = oracle_inputs(p, Y, H, E.DTYPE_BF16)
    want = O.el_layer_step(pr, Yr, Hr, cfg["x"])
    assert rel_err(out, want) <= TOL[1]
    # against the unrounded fp64 problem too (includes input rounding)
    assert rel_err(out, O.el_layer_step(p, Y, H, cfg["x"])) <= TOL[1]


def test_bf16_bart_vs_reference_golden(gpu):
    E = gpu
    g = np.load(GOLD / "step_bart_b2.npz")
    m = json.loads(str(g["meta"]))
    p, Y, H = make_case(m["h"], m["d_m"], m["d_k"], m["n"], m["B"], m["x"], m["param_seed"], m["data_seed"])
    out, layer = run_step(E, p, Y, H, m["x"], E.DTYPE_BF16)
    assert rel_err(out, g["out"]) <= TOL[1]


@pytest.mark.parametrize("n", [1, 7, 33, 64, 127, 130, 1000])
def test_bf16_context_lengths(gpu, n):
    E = gpu
    c = BART_CFG
    p, Y, H = make_case(c["h"], c["d_m"], c["d_k"], n, 2, c["x"], 11, 12 + n)
    out, _ = run_step(E, p, Y, H, c["x"], E.DTYPE_BF16)
    pr, Yr, Hr = oracle_inputs(p, Y, H, E.DTYPE_BF16)
    assert rel_err(out, O.el_layer_step(pr, Yr, Hr, c["x"])) <= TOL[1]


@pytest.mark.parametrize("dtype", [0, 1])
def test_ragged_inputs(gpu, dtype):
    """Per-input context lengths; padded rows of H_b are garbage that must be ignored."""
    E = gpu
    c = dict(BART_CFG) if dtype == 1 else dict(ORACLE_CFG)
    B, n = 4, 300
    p, Y, H = make_case(c["h"], c["d_m"], c["d_k"], n, B, c["x"], 21, 22)
    npi = np.array([300, 1, 129, 64], dtype=np.int32)
    Hg = H.copy()
    for b, nb in enumerate(npi):
        Hg[b, nb:] = 1e4 * (1 + b)  # large garbage beyond n_b
    out, _ = run_step(E, p, Y, Hg, c["x"], dtype, npi)
    pr, Yr, Hr = oracle_inputs(p, Y, H, dtype)
    want = O.el_layer_step(pr, Yr, Hr, c["x"], npi)
    assert np.all(np.isfinite(out))
    assert rel_err(out, want) <= TOL[dtype]


@pytest.mark.parametrize("dtype", [0, 1])
def test_batch_bookkeeping_is_exact(gpu, dtype):
    """Output rows b*x+k depend only on (H_b, Y_{b,k}): permuting inputs permutes rows bit-exactly."""
    E = gpu
    c = BART_CFG if dtype == 1 else ORACLE_CFG
    B = 6
    p, Y, H = make_case(c["h"], c["d_m"], c["d_k"], 257, B, c["x"], 31, 32)
    out, layer = run_step(E, p, Y, H, c["x"], dtype)
    perm = np.array([3, 0, 5, 1, 4, 2])
    Yp = Y.reshape(B, c["x"], -1)[perm].reshape(B * c["x"], -1)
    out2, _ = run_step(E, p, Yp, H[perm], c["x"], dtype)
    assert np.array_equal(out2.reshape(B, c["x"], -1), out.reshape(B, c["x"], -1)[perm])


@pytest.mark.parametrize("c,B,picks", [
    (BART_CFG, 320, (0, 1, 157, 318, 319)),          # config 2 at the bench shape (stream-K / tail-split)
    (TBIG_GREEDY_CFG, 512, (0, 255, 511)),           # config 3: greedy, 16 rows per input
    (BEAM12_CFG, 32, (0, 13, 31)),                   # config 5: beam 12 = 3 virtual 64-row inputs
])
def test_bf16_full_size_strided_subset(gpu, c, B, picks):
    """BASELINE configs 2, 3 and 5 at full batch on the GPU, a strided subset of inputs
    checked against the oracle."""
    E = gpu
    import torch

    p = O.params_random(c["h"], c["d_m"], c["d_k"], O.OracleRng(1))
    gen = torch.Generator(device="cuda").manual_seed(2)
    # 671 MB of H generated in HBM (too large for a host fp64 copy); U(-1, 1)
    Hd = (torch.rand((B, c["n"], c["d_m"]), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
    Yd = (torch.rand((B * c["x"], c["d_m"]), generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16)
    layer = E.ElAttentionLayer(to_prod(p), E.DTYPE_BF16)
    out = layer.step(Yd, Hd).double().cpu().numpy()
    assert np.all(np.isfinite(out))
    pr = round_params(p, E.DTYPE_BF16)
    for b in picks:
        Yb = Yd[b * c["x"]:(b + 1) * c["x"]].double().cpu().numpy()
        Hb = Hd[b:b + 1].double().cpu().numpy()
        want = O.el_layer_step(pr, Yb, Hb, c["x"])
        assert rel_err(out[b * c["x"]:(b + 1) * c["x"]], want) <= TOL[1], b


@pytest.mark.parametrize("npi_mode", [False, True])
def test_decoder_step_graph_matches_layer_chain(gpu, npi_mode):
    """DecoderStep (L layers captured into one CUDA graph) == chaining layer.step L times,
    bit-exactly, on replay after replay; and the 2-layer chain matches the oracle."""
    import torch

    E = gpu
    c = BART_CFG
    B, L, n = 3, 3, 200
    layers = [E.ElAttentionLayer(E.AttentionParams.random(c["h"], c["d_m"], c["d_k"], E.Rng(40 + l)), E.DTYPE_BF16)
              for l in range(L)]
    g = torch.Generator(device="cuda").manual_seed(5)
    H = (torch.rand((B, n, c["d_m"]), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    npi = torch.tensor([200, 17, 130], dtype=torch.int32, device="cuda") if npi_mode else None
    dec = E.DecoderStep(layers, H, B, c["x"], npi)
    assert dec.kernels_per_run >= 2 * L  # q' GEMM and decode per layer (+ merge if split); Q/V/out on cuBLASLt
    for it in range(2):
        Y = (torch.rand((B * c["x"], c["d_m"]), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
        got = dec.run(Y).clone()
        torch.cuda.synchronize()
        y = Y
        for ly in layers:
            y = ly.step(y, H, npi)
        torch.cuda.synchronize()
        assert torch.equal(got, y), it
    # oracle for the first two layers of the chain
    dec2 = E.DecoderStep(layers[:2], H, B, c["x"], npi)
    out = dec2.run(Y).double().cpu().numpy()
    pr = [round_params(O.params_random(c["h"], c["d_m"], c["d_k"], O.OracleRng(40 + l)), E.DTYPE_BF16)
          for l in range(2)]
    from paper_2105_04779_b200.attention import round_to_dtype

    Hh = H.double().cpu().numpy()
    y = Y.double().cpu().numpy()
    nl = npi.cpu().numpy() if npi is not None else None
    for l in range(2):
        y = round_to_dtype(O.el_layer_step(pr[l], y, Hh, c["x"], nl), E.DTYPE_BF16)
    assert rel_err(out, y) <= TOL[1]


@pytest.mark.parametrize("B", [102, 148])
def test_decoder_step_graph_schedules(gpu, B):
    """The decoder step's graph (weights and H fetched before each kernel's PDL wait) is
    bit-identical to the eager layer chain (no early fetches) under the tail-split (B = 102:
    one full round + 28 inputs in 2 parts) and whole-input (B = 148: two full rounds)
    decode schedules."""
    import torch

    E = gpu
    c = BART_CFG
    L, n = 2, 256
    layers = [E.ElAttentionLayer(E.AttentionParams.random(c["h"], c["d_m"], c["d_k"], E.Rng(60 + l)), E.DTYPE_BF16)
              for l in range(L)]
    g = torch.Generator(device="cuda").manual_seed(B)
    H = (torch.rand((B, n, c["d_m"]), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    dec = E.DecoderStep(layers, H, B, c["x"])
    Y = (torch.rand((B * c["x"], c["d_m"]), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    got = dec.run(Y).clone()
    again = dec.run(Y).clone()
    torch.cuda.synchronize()
    y = Y
    for ly in layers:
        y = ly.step(y, H)
    torch.cuda.synchronize()
    assert torch.equal(got, y) and torch.equal(again, y)


@pytest.mark.parametrize("dtype", [0, 1])
def test_hidden_state_cache_self_attention(gpu, dtype):
    """Decoder-only EL self-attention over per-lane hidden-state caches (config 4 form):
    append the lane's input, attend over its history (x = 1, ragged lengths), reorder
    lanes with gather — against the oracle's el_layer_step per lane."""
    import torch

    E = gpu
    c = dict(BART_CFG) if dtype == 1 else dict(ORACLE_CFG)
    lanes, n_max, steps = 6, 40, 5
    p = O.params_random(c["h"], c["d_m"], c["d_k"], O.OracleRng(77))
    layer = E.ElAttentionLayer(to_prod(p), dtype)
    cache = E.HiddenStateCache(1, lanes, n_max, c["d_m"], dtype)
    td = torch.bfloat16 if dtype == 1 else torch.float32
    rng = O.OracleRng(78)
    pr = round_params(p, dtype)
    from paper_2105_04779_b200.attention import round_to_dtype

    hist = [[] for _ in range(lanes)]  # host mirror of each lane's history
    # prefix of different lengths per lane
    for l in range(lanes):
        for _ in range(1 + l):
            y = round_to_dtype(rng.uniform((1, c["d_m"])), dtype)
            hist[l].append(y[0])
    maxlen = max(len(hh) for hh in hist)
    for t in range(maxlen):  # ingest lane by lane at its own pace
        Yt = np.zeros((lanes, c["d_m"]))
        for l in range(lanes):
            if t < len(hist[l]):
                Yt[l] = hist[l][t]
        Ydev = torch.from_numpy(Yt).to("cuda", td)
        # lanes that are done get appended garbage we then truncate by resetting lengths
        cache.append(0, Ydev)
    cache.lengths[0] = torch.tensor([len(hh) for hh in hist], dtype=torch.int32, device="cuda")
    for step in range(steps):
        Y = round_to_dtype(rng.uniform((lanes, c["d_m"])), dtype)
        cache.append(0, torch.from_numpy(Y).to("cuda", td))
        for l in range(lanes):
            hist[l].append(Y[l])
        out = cache.attend(layer, 0, torch.from_numpy(Y).to("cuda", td)).double().cpu().numpy()
        for l in range(lanes):
            Hl = np.stack(hist[l])[None]
            want = O.el_layer_step(pr, Y[l:l + 1], Hl, 1)
            assert rel_err(out[l:l + 1], want) <= TOL[dtype], (step, l)
        parent = [(l * 5 + step) % lanes for l in range(lanes)]  # reorder (parents repeat)
        cache.gather(parent, rows_hint=n_max)
        hist = [list(hist[q]) for q in parent]
        assert cache.lengths[0].cpu().tolist() == [len(hh) for hh in hist]
        got = cache.lane_view(0).double().cpu().numpy()
        for l in range(lanes):
            assert np.array_equal(got[l, :len(hist[l])], np.stack(hist[l]))


@pytest.mark.parametrize("kb,vb,t_out", [(1, 1, 3), (1, 1, 0), (0, 1, 2), (1, 0, 4), (0, 0, 1)])
def test_fp32_mixed_self_attention_vs_oracle(gpu, kb, vb, t_out):
    """Reference-shaped mixed_self_attention (attention.hpp:309-365) on the fp32 path vs the
    oracle (itself pinned bit-exact to the reference in test_oracle.py)."""
    E = gpu
    rng = O.OracleRng(900 + 10 * kb + vb + t_out)
    p = O.params_random(4, 16, 4, rng)
    p.include_key_bias, p.include_value_bias = bool(kb), bool(vb)
    q, Hp, gen = rng.uniform((1, 16)), rng.uniform((5, 16)), rng.uniform((t_out, 16))
    got = E.mixed_self_attention(q, Hp, gen, to_prod(p), E.DTYPE_F32)
    want = O.mixed_self_attention(p, q, Hp, gen)
    assert rel_err(got, want) <= TOL[0]


@pytest.mark.parametrize("dtype", [0, 1])
def test_mixed_self_attention_batched_vs_oracle(gpu, dtype):
    """Batched decoder-only steps: B inputs x x lanes share their input's prefix, each lane
    appends its row to its own generated cache then attends (model.hpp:365-367)."""
    import torch

    E = gpu
    c = dict(BART_CFG) if dtype == 1 else dict(ORACLE_CFG)
    B, x, n, steps = 3, c["x"], 150, 4
    p = O.params_random(c["h"], c["d_m"], c["d_k"], O.OracleRng(501))
    layer = E.ElAttentionLayer(to_prod(p), dtype)
    td = torch.bfloat16 if dtype == 1 else torch.float32
    from paper_2105_04779_b200.attention import round_to_dtype

    rng = O.OracleRng(502)
    P = round_to_dtype(rng.uniform((B, n, c["d_m"])), dtype)
    npi = np.array([150, 33, 97], dtype=np.int32)
    Pd = torch.from_numpy(P).to("cuda", td)
    npd = torch.from_numpy(npi).cuda()
    cache = E.KvCache(layer, B * x, steps)
    pr = round_params(p, dtype)
    gen = [[] for _ in range(B * x)]
    for step in range(steps):
        Y = round_to_dtype(rng.uniform((B * x, c["d_m"])), dtype)
        Yd = torch.from_numpy(Y).to("cuda", td)
        cache.append(Yd)
        for r in range(B * x):
            gen[r].append(Y[r])
        out = E.mixed_self_attention_batched(layer, Yd, Pd, cache, x, npd).double().cpu().numpy()
        for r in range(B * x):
            b = r // x
            want = O.mixed_self_attention(pr, Y[r:r + 1], P[b, :npi[b]], np.stack(gen[r]))
            assert rel_err(out[r:r + 1], want) <= TOL[dtype], (step, r)


def test_mixed_self_attention_split_prefixes_vs_oracle(gpu):
    """The decode's softmax statistics {m, l} when inputs are split across clusters: 24 inputs
    with full 1024-row prefixes run as 3 parts each (tail-split with no full round), merged by
    the merge kernel, which also emits the statistics the mixed combine consumes."""
    import torch

    E = gpu
    c = dict(BART_CFG)
    B, x, n = 24, c["x"], 1024
    p = O.params_random(c["h"], c["d_m"], c["d_k"], O.OracleRng(511))
    layer = E.ElAttentionLayer(to_prod(p), E.DTYPE_BF16)
    from paper_2105_04779_b200.attention import round_to_dtype

    g = torch.Generator(device="cuda").manual_seed(512)
    Pd = (torch.rand((B, n, c["d_m"]), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    Yd = (torch.rand((B * x, c["d_m"]), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    cache = E.KvCache(layer, B * x, 2)
    cache.append(Yd)
    out = E.mixed_self_attention_batched(layer, Yd, Pd, cache, x, None).double().cpu().numpy()
    pr = round_params(p, E.DTYPE_BF16)
    Y = Yd.double().cpu().numpy()
    for r in (0, 5, 47, 95):
        b = r // x
        want = O.mixed_self_attention(pr, Y[r:r + 1], Pd[b].double().cpu().numpy(), Y[r:r + 1])
        assert rel_err(out[r:r + 1], want) <= TOL[1], r


@pytest.mark.parametrize("h,d_m", [(4, 256), (12, 768)])
def test_bf16_step_other_model_widths(gpu, h, d_m):
    """d_m = 256 / 768 (UNITS = 1 / 3 of the tcgen05 decode), beam 4 and greedy."""
    E = gpu
    for x in (4, 1):
        p, Y, H = make_case(h, d_m, 64, 300, 3, x, 81 + h, 82 + x)
        out, layer = run_step(E, p, Y, H, x, E.DTYPE_BF16)
        assert layer.dev.decode_kernel_kind(x) == 1
        pr, Yr, Hr = oracle_inputs(p, Y, H, E.DTYPE_BF16)
        assert rel_err(out, O.el_layer_step(pr, Yr, Hr, x)) <= TOL[1], (h, d_m, x)


# ---------------------------------------------------------------- beam-search candidates
def _beam_check(E, lp, live, lanes, k, roots, pen=None):
    import torch

    B, V = lp.shape[0] // lanes, lp.shape[1]
    par, tok, lps = E.beam_candidates(torch.from_numpy(lp).float().cuda(), torch.from_numpy(live).float().cuda(),
                                      lanes, k, roots,
                                      penalty=torch.from_numpy(pen).float().cuda() if pen is not None else None)
    torch.cuda.synchronize()
    par, tok, lps = par.cpu().numpy(), tok.cpu().numpy(), lps.cpu().numpy()
    for b in range(B):
        ep, et, el = O.beam_candidates(lp[b * lanes:(b + 1) * lanes], live[b * lanes:(b + 1) * lanes], k, roots,
                                       penalty=pen[b] if pen is not None else None)
        assert np.array_equal(par[b], ep) and np.array_equal(tok[b], et), (b, par[b], ep, tok[b], et)
        assert np.array_equal(lps[b].astype(np.float64), el)


def test_beam_candidates_golden_gpu(gpu):
    """Device candidate selection vs the reference's own order (decoding.hpp:163-205)."""
    import torch

    E = gpu
    g = np.load(GOLD / "beam_candidates.npz")
    k = int(g["k"])
    for b in range(g["lprobs"].shape[0]):
        lp, live = g["lprobs"][b], g["live"][b]
        par, tok, lps = E.beam_candidates(torch.from_numpy(lp).float().cuda(), torch.from_numpy(live).float().cuda(),
                                          lp.shape[0], k, int(g["roots"][b]))
        assert np.array_equal(par.cpu().numpy()[0], g["parent"][b])
        assert np.array_equal(tok.cpu().numpy()[0], g["token"][b])
        assert np.array_equal(lps.cpu().numpy()[0].astype(np.float64), g["lp_sum"][b])
        par, tok, lps = E.beam_candidates(torch.from_numpy(lp).float().cuda(), torch.from_numpy(live).float().cuda(),
                                          lp.shape[0], k, int(g["roots"][b]),
                                          penalty=torch.from_numpy(g["penalty"][b][None]).float().cuda())
        assert np.array_equal(par.cpu().numpy()[0], g["parent_pen"][b])
        assert np.array_equal(tok.cpu().numpy()[0], g["token_pen"][b])
        assert np.array_equal(lps.cpu().numpy()[0].astype(np.float64), g["lp_sum_pen"][b])


@pytest.mark.parametrize("lanes,V,k,roots", [(4, 50265, 8, 4), (4, 50265, 8, 1), (12, 50265, 24, 12),
                                             (5, 1000, 32, 3), (1, 7, 10, 1), (8, 3, 32, 8)])
def test_beam_candidates_vs_oracle(gpu, lanes, V, k, roots):
    """BART-vocabulary candidate selection; values on a 1/8 grid (ties, exact fp32 sums),
    masked (-inf) tokens, fewer finite candidates than k where V*roots is small."""
    E = gpu
    rng = np.random.default_rng(lanes * 1000 + V + k)
    B = 3
    lp = np.round(rng.uniform(-30, 0, (B * lanes, V)) * 8) / 8
    lp[rng.random(lp.shape) < 0.05] = -np.inf
    lp[0, :] = -np.inf  # a fully masked parent
    live = np.round(rng.uniform(-10, 0, B * lanes) * 8) / 8
    _beam_check(E, lp, live, lanes, k, roots)


def test_beam_candidates_diverse_penalty(gpu):
    """Diverse beam search: per-input token penalties strength x counts subtracted before the
    sum (decoding.hpp:312-316), BART vocabulary, ties on the 1/8 grid."""
    E = gpu
    rng = np.random.default_rng(77)
    B, lanes, V, k = 4, 3, 50265, 6
    lp = np.round(rng.uniform(-20, 0, (B * lanes, V)) * 8) / 8
    lp[rng.random(lp.shape) < 0.05] = -np.inf
    live = np.round(rng.uniform(-6, 0, B * lanes) * 8) / 8
    pen = 0.5 * rng.integers(0, 3, (B, V)).astype(np.float64)
    _beam_check(E, lp, live, lanes, k, lanes, pen)


def test_lane_bookkeeping_on_device(gpu):
    """gather (resize) / keep / permute of both cache kinds match the same index operation on
    the host copies (model.hpp:291-325); device parents out of range give NaN lanes."""
    import torch

    E = gpu
    c = BART_CFG
    p = E.AttentionParams.random(4, 256, 64, E.Rng(9))
    layer = E.ElAttentionLayer(p, E.DTYPE_BF16)
    g = torch.Generator(device="cuda").manual_seed(2)
    # hidden-state cache: 2 layers, 4 lanes, ragged lengths
    hc = E.HiddenStateCache(2, 4, 16, 256, E.DTYPE_BF16)
    hc.cache.copy_((torch.rand(hc.cache.shape, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16))
    hc.lengths.copy_(torch.tensor([[3, 16, 7, 1], [2, 5, 9, 16]], dtype=torch.int32))
    ref_c, ref_l = hc.cache.clone(), hc.lengths.clone()
    hc.gather([1, 1, 3, 0, 2])  # expansion to 5 lanes
    idx = torch.tensor([1, 1, 3, 0, 2], device="cuda")
    assert torch.equal(hc.lengths, ref_l[:, idx])
    for l in range(2):
        for i, pi in enumerate([1, 1, 3, 0, 2]):
            n = int(ref_l[l, pi])
            assert torch.equal(hc.lane_view(l)[i, :n], ref_c[l, pi, :n])
    hc.keep([True, False, True, True, False])
    assert hc.lanes == 3 and torch.equal(hc.lengths, ref_l[:, torch.tensor([1, 3, 0], device="cuda")])
    hc.permute([2, 0, 1])
    assert torch.equal(hc.lengths, ref_l[:, torch.tensor([0, 1, 3], device="cuda")])
    with pytest.raises(E.StateError):
        hc.keep([False, False, False])
    # mixed-form K/V cache
    kv = E.KvCache(layer, 4, 8)
    kv.K.copy_((torch.rand(kv.K.shape, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16))
    kv.V.copy_((torch.rand(kv.V.shape, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16))
    K0, V0 = kv.K.clone(), kv.V.clone()
    kv.gather([3, 3, 1])
    sel = torch.tensor([3, 3, 1], device="cuda")
    assert kv.R == 3 and torch.equal(kv.K, K0[sel]) and torch.equal(kv.V, V0[sel])
    kv.keep([False, True, True])
    assert torch.equal(kv.K, K0[torch.tensor([3, 1], device="cuda")])
    kv.gather(torch.tensor([0, 7], dtype=torch.int32, device="cuda"))  # device parent 7 is out of range
    torch.cuda.synchronize()
    assert torch.isnan(kv.K[1].float()).all() and torch.equal(kv.K[0], K0[3])


@pytest.mark.parametrize("dtype", [1, 0])
def test_hidden_state_cache_copy_on_fork(gpu, dtype):
    """The slot-indexed cache's fork against a host mirror of gather_lanes (model.hpp:
    291-306) over several reorders: random parents (repeats and drops), a permutation (no
    slot changes hands... every lane keeps its parent's slot), an expansion past the slot
    count (the store grows), an out-of-range device parent (loud length n_max + 1); and the
    attention read through the slot map equals the step over a physically gathered H."""
    import torch

    E = gpu
    L, lanes, n_max, d_m = 2, 6, 24, 256
    td = torch.bfloat16 if dtype == 1 else torch.float32
    g = torch.Generator(device="cuda").manual_seed(5)
    hc = E.HiddenStateCache(L, lanes, n_max, d_m, dtype)
    hc.cache.copy_((torch.rand(hc.cache.shape, generator=g, device="cuda") * 2 - 1).to(td))
    lens = torch.randint(1, n_max, (L, lanes), generator=g, device="cuda", dtype=torch.int32)
    hc.lengths.copy_(lens)
    mirror = [[hc.cache[l, i, : int(lens[l, i])].clone() for i in range(lanes)] for l in range(L)]
    rng = np.random.default_rng(11)
    plans = [list(rng.integers(0, lanes, lanes)), list(rng.permutation(lanes)), list(rng.integers(0, lanes, 4)),
             [0, 1, 1, 2, 3, 3, 3, 0], list(rng.integers(0, 8, 8))]
    for parent in plans:
        slots_before = hc.lane_slot.clone()
        hc.gather([int(p) for p in parent], rows_hint=n_max)
        if sorted(parent) == list(range(len(parent))):  # permutation: histories change lanes, not slots
            assert sorted(hc.lane_slot.tolist()) == sorted(slots_before.tolist())
        mirror = [[mirror[l][int(p)] for p in parent] for l in range(L)]
        assert hc.lanes == len(parent)
        for l in range(L):
            view = hc.lane_view(l)
            for i in range(hc.lanes):
                n = mirror[l][i].shape[0]
                assert int(hc.lengths[l, i]) == n
                assert torch.equal(view[i, :n], mirror[l][i])
        assert len(set(hc.lane_slot.tolist())) == hc.lanes  # every lane owns its slot
    # attention through the slot map == the step over the lane-ordered copy
    p = E.AttentionParams.random(4, d_m, 64, E.Rng(3))
    layer = E.ElAttentionLayer(p, dtype)
    Y = (torch.rand((hc.lanes, d_m), generator=g, device="cuda") * 2 - 1).to(td)
    got = hc.attend(layer, 1, Y)
    want = layer.step(Y, hc.lane_view(1), hc.lengths[1].clone())
    torch.cuda.synchronize()
    assert torch.equal(got, want)
    # out-of-range device parent: loud length, the other lanes intact
    hc.gather(torch.tensor([1, 99], dtype=torch.int32, device="cuda"))
    torch.cuda.synchronize()
    assert int(hc.lengths[0, 1]) == n_max + 1 and int(hc.lengths[0, 0]) == mirror[0][1].shape[0]
    assert torch.equal(hc.lane_view(0)[0, : mirror[0][1].shape[0]], mirror[0][1])


def test_hidden_state_cache_fork_many_lanes(gpu):
    """Copy-on-fork plan over more lanes / slots than one CTA has threads (1300 lanes,
    1500 slots: the plan kernel's strided scans), shrinking and growing lane counts."""
    import torch

    E = gpu
    L, lanes, n_max, d_m = 1, 1300, 6, 256
    g = torch.Generator(device="cuda").manual_seed(9)
    hc = E.HiddenStateCache(L, lanes, n_max, d_m, E.DTYPE_BF16, slots=1500)
    hc.cache.copy_((torch.rand(hc.cache.shape, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16))
    hc.lengths.copy_(torch.randint(1, n_max + 1, (L, lanes), generator=g, device="cuda", dtype=torch.int32))
    view, lens = hc.lane_view(0).clone(), hc.lengths[0].clone()
    rng = np.random.default_rng(4)
    for lanes_out in (1300, 900, 1500):
        parent = rng.integers(0, hc.lanes, lanes_out)
        hc.gather([int(p) for p in parent])
        idx = torch.from_numpy(parent).cuda().long()
        view, lens = view[idx], lens[idx]
        assert torch.equal(hc.lengths[0], lens)
        got = hc.lane_view(0)
        mask = torch.arange(n_max, device="cuda")[None, :] < lens[:, None].long()
        assert torch.equal(got[mask], view[mask])
        assert len(set(hc.lane_slot.tolist())) == hc.lanes


def test_beam_candidates_errors_and_edges(gpu):
    """Reference-style errors at the boundary (k outside [1, 32], roots > lanes, shape
    mismatch) and edges: fewer finite candidates than k (parent -1 rows), V = 1, 256 lanes."""
    import torch

    E = gpu
    lp = torch.zeros(4, 10, device="cuda")
    live = torch.zeros(4, device="cuda")
    with pytest.raises(E.UnsupportedError):
        E.beam_candidates(lp, live, 2, 33)
    with pytest.raises(E.ParamError):
        E.beam_candidates(lp, live, 2, 0)
    with pytest.raises(E.ShapeError):
        E.beam_candidates(lp, live, 2, 4, roots=3)
    with pytest.raises(E.ShapeError):
        E.beam_candidates(lp, live[:3], 2, 4)
    # only 3 finite candidates for k = 5
    lp = torch.full((2, 4), float("-inf"), device="cuda")
    lp[0, 1], lp[0, 3], lp[1, 2] = -1.0, -2.0, -0.5
    par, tok, lps = E.beam_candidates(lp, torch.tensor([0.0, -1.0], device="cuda"), 2, 5)
    # candidates (parent, token, lp_sum): (0, 1, -1.0), (1, 2, -1.5), (0, 3, -2.0)
    assert par.cpu().tolist() == [[0, 1, 0, -1, -1]] and tok.cpu().tolist() == [[1, 2, 3, -1, -1]]
    assert lps.cpu()[0, :3].tolist() == [-1.0, -1.5, -2.0] and torch.isinf(lps.cpu()[0, 3:]).all()
    # V = 1 and 256 lanes
    rng = np.random.default_rng(5)
    lp1 = np.round(rng.uniform(-4, 0, (512, 1)) * 8) / 8
    live1 = np.round(rng.uniform(-4, 0, 512) * 8) / 8
    _beam_check(E, lp1, live1, 256, 16, 256)


def test_fp32_decoder_step_graph_with_split_simt_decode(gpu):
    """fp32 layers in the CUDA-graph decoder step: at the oracle config the SIMT decode splits
    the context over CTAs (stream-ordered scratch inside the capture) — the graph equals
    the eager layer chain."""
    import torch

    E = gpu
    h, d_m, d_k, x, n, B, L = 8, 512, 64, 4, 128, 2, 3
    layers = [E.ElAttentionLayer(E.AttentionParams.random(h, d_m, d_k, E.Rng(10 + l)), E.DTYPE_F32) for l in range(L)]
    g = torch.Generator(device="cuda").manual_seed(1)
    H = torch.rand((B, n, d_m), generator=g, device="cuda") * 2 - 1
    Y = torch.rand((B * x, d_m), generator=g, device="cuda") * 2 - 1
    dec = E.DecoderStep(layers, H, B, x)
    got = dec.run(Y).clone()
    torch.cuda.synchronize()
    y = Y
    for ly in layers:
        y = ly.step(y, H)
    torch.cuda.synchronize()
    assert (got - y).abs().max().item() / y.abs().max().item() < 1e-6
