"""Generate tests/golden/*.npz from the REFERENCE itself.

Runs in the build container only (needs oracle/_ref/libelattn_ref.so, compiled
read-only from /root/reference/proj/include by oracle/Makefile).  Every output
array is produced by the reference's own functions (build_el_query,
el_attention, el_attention_folded, multi_head_attention and the
build_el_query x beams -> fold_el_queries -> el_attention_folded chain).
Inputs are regenerated from seeds by the tests (SplitMix64 is pinned by the
known-answer test), except where noted; small input arrays are stored too.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import oracle as O  # noqa: E402
from cases import ORACLE_CFG, BART_CFG, make_case  # noqa: E402

OUT = Path(__file__).resolve().parent


def ref_case_sweep():
    """test_attention.cpp:230-247 — EL == MHA over 72 configs, Rng(1000 + case_id):
    params = random(h, d_m, d_k, rng); q = U(-1,1)[1, d_m]; H = U(-1,1)[n, d_m]."""
    rows = []
    el_out, mha_out = [], []
    cid = 0
    for h in (1, 2, 4):
        for d_m in (8, 16, 32):
            for d_k in (d_m // h, 3):
                for n in (1, 2, 7, 33):
                    rng = O.OracleRng(1000 + cid)
                    p = O.params_random(h, d_m, d_k, rng)
                    q = rng.uniform((1, d_m))
                    H = rng.uniform((n, d_m))
                    assert np.array_equal(O.ref_params_random(h, d_m, d_k, 1000 + cid).Wq, p.Wq)
                    el_out.append(O.el_attention(p, q, H, impl="reference").ravel())
                    mha_out.append(O.multi_head_attention(p, q, H, impl="reference").ravel())
                    rows.append((1000 + cid, h, d_m, d_k, n))
                    cid += 1
    np.savez_compressed(OUT / "sweep_el_mha.npz", cases=np.array(rows, dtype=np.int64),
                        el=np.concatenate(el_out), mha=np.concatenate(mha_out))
    return {"sweep_el_mha.npz": f"{cid} configs of test_attention.cpp:230-247 (el_attention, multi_head_attention)"}


def ref_case_folded():
    """test_attention.cpp:301-325 — params Rng(71) random(4,16,4); H = random_tensor({9,16},72);
    q_b = random_tensor({1,16}, 80+b)."""
    p = O.params_random(4, 16, 4, O.OracleRng(71))
    H = O.OracleRng(72).uniform((9, 16))
    qs = [O.OracleRng(80 + b).uniform((1, 16)) for b in range(4)]
    elqs, ss = zip(*[O.build_el_query(p, q, impl="reference") for q in qs])
    Q, S = np.concatenate(elqs), np.concatenate(ss)
    folded = O.el_attention_folded(p, Q, H, S, impl="reference")
    singles = np.concatenate([O.el_attention(p, q, H, impl="reference") for q in qs])
    np.savez_compressed(OUT / "folded_g4.npz", H=H, q=np.concatenate(qs), elq=Q, s=S, folded=folded,
                        singles=singles)
    return {"folded_g4.npz": "test_attention.cpp:301-325 (build_el_query, fold, el_attention_folded)"}


def ref_case_build_query():
    """test_attention.cpp:206-227 — params Rng(53) random(3,12,4); q = random_tensor({1,12},54)."""
    p = O.params_random(3, 12, 4, O.OracleRng(53))
    q = O.OracleRng(54).uniform((1, 12))
    elq, s = O.build_el_query(p, q, impl="reference")
    np.savez_compressed(OUT / "build_el_query.npz", q=q, elq=elq, s=s)
    return {"build_el_query.npz": "test_attention.cpp:206-227"}


def ref_case_step(name, cfg, B, param_seed=1, data_seed=2):
    """Batched layer step through the reference chain (SURVEY.md §8 math contract)."""
    p, Y, H = make_case(cfg["h"], cfg["d_m"], cfg["d_k"], cfg["n"], B, cfg["x"], param_seed, data_seed)
    out = O.el_layer_step(p, Y, H, cfg["x"], impl="reference", nthreads=8)
    meta = dict(cfg, B=B, param_seed=param_seed, data_seed=data_seed)
    np.savez_compressed(OUT / f"{name}.npz", out=out, meta=json.dumps(meta))
    return {f"{name}.npz": f"reference layer step, {meta}"}


def beam_inputs(seed=7):
    """Beam candidate inputs: lanes 4, V 97, log-probs on a 1/4 grid (ties on purpose, exact
    sums in fp32) with ~10% -inf (masked tokens); three inputs with roots 1, 4, 3."""
    rng = np.random.default_rng(seed)
    lp = np.round(rng.uniform(-6, 0, (3, 4, 97)) * 4) / 4
    lp[rng.random(lp.shape) < 0.1] = -np.inf
    live = np.round(rng.uniform(-4, 0, (3, 4)) * 4) / 4
    return lp, live, (1, 4, 3), 10


def ref_case_beam():
    """decoding.hpp:186-205 candidate generation + candidate_better (:163-167) order."""
    lp, live, roots, k = beam_inputs()
    outs = [O.beam_candidates(lp[b], live[b], k, roots[b], impl="reference") for b in range(3)]
    # diverse-beam token penalties (strength 0.5 x counts 0..2, decoding.hpp:312-316)
    pen = 0.5 * np.random.default_rng(8).integers(0, 3, (3, lp.shape[2])).astype(np.float64)
    outp = [O.beam_candidates(lp[b], live[b], k, roots[b], impl="reference", penalty=pen[b]) for b in range(3)]
    np.savez_compressed(OUT / "beam_candidates.npz", lprobs=lp, live=live, roots=np.array(roots), k=k,
                        parent=np.stack([o[0] for o in outs]), token=np.stack([o[1] for o in outs]),
                        lp_sum=np.stack([o[2] for o in outs]), penalty=pen,
                        parent_pen=np.stack([o[0] for o in outp]), token_pen=np.stack([o[1] for o in outp]),
                        lp_sum_pen=np.stack([o[2] for o in outp]))
    return {"beam_candidates.npz": "beam_search candidates, decoding.hpp:186-205 (order :163-167); "
                                   "*_pen: with diverse-beam token penalties (:312-316)"}


def main():
    if not O.ref_available():
        raise SystemExit("oracle/_ref not built: run `make -C oracle` with /root/reference present")
    kat = np.array([O.ref_lib().ref_rng_first(s, k) for s in (0, 1, 42) for k in range(4)], dtype=np.uint64)
    np.savez_compressed(OUT / "rng_kat.npz", seeds=np.array([0, 1, 42]), first4=kat.reshape(3, 4))
    manifest = {"rng_kat.npz": "SplitMix64 first 4 outputs for seeds 0,1,42 (tensor.hpp:133-150)"}
    manifest.update(ref_case_sweep())
    manifest.update(ref_case_folded())
    manifest.update(ref_case_build_query())
    manifest.update(ref_case_step("step_oracle_cfg", ORACLE_CFG, ORACLE_CFG["B"]))
    manifest.update(ref_case_step("step_bart_b2", BART_CFG, 2))
    manifest.update(ref_case_beam())
    (OUT / "MANIFEST.json").write_text(json.dumps(manifest, indent=2) + "\n")
    print(json.dumps(manifest, indent=2))


if __name__ == "__main__":
    main()
