"""Pins the oracle (oracle/elattn_oracle.c) before anything is checked against it.

1. Golden vectors produced by the reference itself (tests/golden, make_golden.py).
2. The reference's own known-answer tests for this path, restated
   (test_tensor.cpp:165-170, test_attention.cpp:120-130, 189-331).
3. The product's host-side RNG / parameter layout against the oracle's.
"""
import json
from pathlib import Path

import numpy as np
import pytest

import oracle as O
from cases import ORACLE_CFG, BART_CFG, make_case, rel_err

GOLD = Path(__file__).resolve().parent / "golden"


def identity_params(d_m):
    """test_attention.cpp:16-30."""
    I = np.eye(d_m)[None]
    z = np.zeros((1, d_m))
    return O.Params(1, d_m, d_m, I.copy(), I.copy(), I.copy(), I.copy(), z.copy(), z.copy(), z.copy(),
                    np.zeros(d_m))


def test_splitmix64_known_answer():
    # test_tensor.cpp:165-170 — published SplitMix64 fixed point.
    r = O.OracleRng(0)
    assert r.next_u64() == 0xE220A8397B1DCDAF
    assert r.next_u64() == 0x6E789E6AA1B965F4
    g = np.load(GOLD / "rng_kat.npz")
    for seed, want in zip(g["seeds"], g["first4"]):
        r = O.OracleRng(int(seed))
        assert [r.next_u64() for _ in range(4)] == [int(v) for v in want]


def test_product_rng_matches_oracle():
    from paper_2105_04779_b200.attention import AttentionParams, Rng, seeded_uniform

    r = Rng(0)
    assert r.next_u64() == 0xE220A8397B1DCDAF and r.next_u64() == 0x6E789E6AA1B965F4
    p = AttentionParams.random(3, 24, 5, Rng(99))
    q = O.params_random(3, 24, 5, O.OracleRng(99))
    for name in ("Wq", "Wk", "Wv", "Wo", "bq", "bk", "bv", "bo"):
        assert np.array_equal(getattr(p, name), getattr(q, name)), name
    a = seeded_uniform((7, 5), Rng(3), -1, 1)
    assert np.array_equal(a, O.OracleRng(3).uniform((7, 5)))


def test_sweep_el_equals_mha_golden():
    """test_attention.cpp:230-247: 72 configs; port must reproduce the reference bit-for-bit."""
    g = np.load(GOLD / "sweep_el_mha.npz")
    off = 0
    worst_el_mha = 0.0
    for seed, h, d_m, d_k, n in g["cases"]:
        rng = O.OracleRng(int(seed))
        p = O.params_random(int(h), int(d_m), int(d_k), rng)
        q = rng.uniform((1, int(d_m)))
        H = rng.uniform((int(n), int(d_m)))
        el = O.el_attention(p, q, H).ravel()
        mha = O.multi_head_attention(p, q, H).ravel()
        assert np.array_equal(el, g["el"][off:off + d_m])
        assert np.array_equal(mha, g["mha"][off:off + d_m])
        worst_el_mha = max(worst_el_mha, np.max(np.abs(el - mha)))
        off += int(d_m)
    assert worst_el_mha <= 1e-10  # the reference's own gate


def test_folded_golden():
    g = np.load(GOLD / "folded_g4.npz")
    p = O.params_random(4, 16, 4, O.OracleRng(71))
    assert np.array_equal(O.OracleRng(72).uniform((9, 16)), g["H"])
    elqs, ss = zip(*[O.build_el_query(p, g["q"][b:b + 1]) for b in range(4)])
    Q, S = np.concatenate(elqs), np.concatenate(ss)
    assert np.array_equal(Q, g["elq"]) and np.array_equal(S, g["s"])
    folded = O.el_attention_folded(p, Q, g["H"], S)
    assert np.array_equal(folded, g["folded"])
    # g=4 equals four independent el_attention calls (test_attention.cpp:313-325)
    assert np.max(np.abs(folded - g["singles"])) <= 1e-12


def test_build_el_query_golden():
    g = np.load(GOLD / "build_el_query.npz")
    p = O.params_random(3, 12, 4, O.OracleRng(53))
    elq, s = O.build_el_query(p, g["q"])
    assert np.array_equal(elq, g["elq"]) and np.array_equal(s, g["s"])
    # explicit product oracle (test_attention.cpp:206-227)
    for i in range(3):
        Qi = g["q"][0] @ p.Wq[i] + p.bq[i]
        assert np.max(np.abs(elq[i] - Qi @ p.Wk[i].T)) <= 1e-12
        assert abs(s[i] - Qi @ p.bk[i]) <= 1e-12


@pytest.mark.parametrize("name", ["step_oracle_cfg", "step_bart_b2"])
def test_layer_step_golden(name):
    g = np.load(GOLD / f"{name}.npz")
    meta = json.loads(str(g["meta"]))
    p, Y, H = make_case(meta["h"], meta["d_m"], meta["d_k"], meta["n"], meta["B"], meta["x"],
                        meta["param_seed"], meta["data_seed"])
    out = O.el_layer_step(p, Y, H, meta["x"])
    assert np.array_equal(out, g["out"])


def test_known_answers():
    # identity weights, zero biases, zero query: row mean of H (test_attention.cpp:250-259)
    p = identity_params(4)
    H = O.OracleRng(61).uniform((5, 4))
    out = O.el_attention(p, np.zeros((1, 4)), H)
    assert np.max(np.abs(out[0] - H.mean(axis=0))) <= 1e-12
    # n = 1 returns the (projected) single row: identity params -> H row (test_attention.cpp:92-98)
    H1 = O.OracleRng(7).uniform((1, 4))
    assert np.max(np.abs(O.el_attention(p, O.OracleRng(5).uniform((1, 4)), H1) - H1)) <= 1e-15
    # key-bias flag does not change the output (test_attention.cpp:260-271)
    p2 = O.params_random(2, 8, 4, O.OracleRng(62))
    q, Hk = O.OracleRng(63).uniform((1, 8)), O.OracleRng(64).uniform((6, 8))
    with_kb = O.el_attention(p2, q, Hk)
    p2.include_key_bias = False
    assert np.max(np.abs(with_kb - O.el_attention(p2, q, Hk))) <= 1e-12


def test_errors_mirror_reference():
    p = O.params_random(4, 16, 4, O.OracleRng(71))
    H = O.OracleRng(72).uniform((9, 16))
    with pytest.raises(O.OracleError) as e:  # rows not divisible by h (test_attention.cpp:326-330)
        O.el_attention_folded(p, O.OracleRng(90).uniform((6, 16)), H, np.zeros(6))
    assert e.value.status == 1
    with pytest.raises(O.OracleError) as e:  # empty context (test_attention.cpp:294-298)
        O.el_attention(p, np.zeros((1, 16)), np.zeros((0, 16)))
    assert e.value.status == 3
    if O.ref_available():
        for impl in ("port", "reference"):
            with pytest.raises(O.OracleError) as e:
                O.el_attention_folded(p, O.OracleRng(90).uniform((6, 16)), H, np.zeros(6), impl=impl)
            assert e.value.status == 1


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built here")
def test_port_equals_reference_random():
    """Port vs the compiled reference on fresh random shapes (incl. ragged n per input)."""
    for seed, (h, d_m, d_k, n, B, x) in enumerate([(2, 16, 8, 5, 3, 2), (4, 32, 3, 17, 2, 3), (8, 64, 8, 33, 2, 4)]):
        p, Y, H = make_case(h, d_m, d_k, n, B, x, 100 + seed, 200 + seed)
        npi = np.array([n - i for i in range(B)], dtype=np.int32)
        a = O.el_layer_step(p, Y, H, x, npi)
        b = O.el_layer_step(p, Y, H, x, npi, impl="reference", nthreads=2)
        assert np.array_equal(a, b)
        assert rel_err(a, b) == 0.0


@pytest.mark.parametrize("kb,vb,t_out", [(1, 1, 3), (1, 1, 0), (0, 1, 2), (1, 0, 4), (0, 0, 1)])
def test_mixed_self_attention_and_kv_cache_match_reference(kb, vb, t_out):
    """Decoder-only path: KvCache::append (attention.hpp:134-150) and mixed_self_attention
    (:309-365) restated in the oracle == the reference's own functions, bit for bit."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built (reference headers absent)")
    rng = O.OracleRng(900 + 10 * kb + vb + t_out)
    p = O.params_random(4, 16, 4, rng)
    p.include_key_bias, p.include_value_bias = bool(kb), bool(vb)
    q = rng.uniform((1, 16))
    Hp = rng.uniform((5, 16))
    gen = rng.uniform((t_out, 16))
    K, V = O.kv_build(p, gen, t_max=max(t_out, 1))
    Kr, Vr = O.kv_build(p, gen, t_max=max(t_out, 1), impl="reference")
    assert np.array_equal(K, Kr) and np.array_equal(V, Vr)
    out = O.mixed_self_attention(p, q, Hp, gen)
    ref = O.mixed_self_attention(p, q, Hp, gen, impl="reference")
    assert np.array_equal(out, ref)


def test_mixed_self_attention_reduces_to_el_attention_without_cache():
    """t_out = 0: the joint softmax is the prefix softmax, so mixed == el_attention."""
    rng = O.OracleRng(950)
    p = O.params_random(2, 8, 4, rng)
    q, Hp = rng.uniform((1, 8)), rng.uniform((6, 8))
    a = O.mixed_self_attention(p, q, Hp, np.zeros((0, 8)))
    b = O.el_attention(p, q, Hp)
    assert np.max(np.abs(a - b)) <= 1e-12


def test_beam_candidates_golden():
    """Port of beam_search's candidate order vs the reference's own (decoding.hpp:163-205)."""
    g = np.load(GOLD / "beam_candidates.npz")
    k = int(g["k"])
    for b in range(g["lprobs"].shape[0]):
        par, tok, lps = O.beam_candidates(g["lprobs"][b], g["live"][b], k, int(g["roots"][b]))
        assert np.array_equal(par, g["parent"][b]) and np.array_equal(tok, g["token"][b])
        assert np.array_equal(lps, g["lp_sum"][b])
        par, tok, lps = O.beam_candidates(g["lprobs"][b], g["live"][b], k, int(g["roots"][b]), penalty=g["penalty"][b])
        assert np.array_equal(par, g["parent_pen"][b]) and np.array_equal(tok, g["token_pen"][b])
        assert np.array_equal(lps, g["lp_sum_pen"][b])


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built here")
def test_beam_candidates_port_equals_reference_random():
    rng = np.random.default_rng(11)
    for _ in range(25):
        lanes, V, k = int(rng.integers(1, 9)), int(rng.integers(1, 300)), int(rng.integers(1, 33))
        roots = int(rng.integers(1, lanes + 1))
        lp = np.round(rng.uniform(-8, 0, (lanes, V)) * 4) / 4
        lp[rng.random((lanes, V)) < 0.2] = -np.inf
        live = np.round(rng.uniform(-5, 0, lanes) * 4) / 4
        pen = 0.25 * rng.integers(0, 4, V) if rng.random() < 0.5 else None
        a = O.beam_candidates(lp, live, k, roots, penalty=pen)
        b = O.beam_candidates(lp, live, k, roots, impl="reference", penalty=pen)
        assert all(np.array_equal(x, y) for x, y in zip(a, b))
