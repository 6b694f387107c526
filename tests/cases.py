"""Seeded synthetic cases shared by the tests, smoke() and the golden script.

Input protocol: weights from ``AttentionParams::random``
(U(-0.1, 0.1), attention.hpp:53-80) driven by SplitMix64 seeded with
``param_seed``; activations U(-1, 1) from a second SplitMix64 seeded with
``data_seed``: first H [B, n, d_m], then Y [B*x, d_m].  Generated with the
oracle's RNG (oracle/liboracle.so), which is pinned to the reference by the
SplitMix64 known-answer test.
"""
from __future__ import annotations

import numpy as np

import oracle as O

# BASELINE.json configs (the hot-path shapes)
ORACLE_CFG = dict(h=8, d_m=512, d_k=64, n=128, B=2, x=4)          # configs[0], fp32
BART_CFG = dict(h=16, d_m=1024, d_k=64, n=1024, x=4)               # configs[1], B 32..320, bf16
TBIG_GREEDY_CFG = dict(h=16, d_m=1024, d_k=64, n=512, x=1)         # configs[2]
BEAM12_CFG = dict(h=16, d_m=1024, d_k=64, n=1024, x=12)            # configs[4]


def make_params(h, d_m, d_k, param_seed):
    return O.params_random(h, d_m, d_k, O.OracleRng(param_seed))


def make_data(B, x, n, d_m, data_seed):
    rng = O.OracleRng(data_seed)
    H = rng.uniform((B, n, d_m), -1.0, 1.0)
    Y = rng.uniform((B * x, d_m), -1.0, 1.0)
    return Y, H


def make_case(h, d_m, d_k, n, B, x, param_seed=1, data_seed=2):
    p = make_params(h, d_m, d_k, param_seed)
    Y, H = make_data(B, x, n, d_m, data_seed)
    return p, Y, H


def rel_err(got, want) -> float:
    """max_abs_diff(got, want) / max|want| (tensor.hpp:287-293, normalised)."""
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    return float(np.max(np.abs(got - want)) / max(np.max(np.abs(want)), 1e-300))


def round_params(p, dtype):
    """Weights rounded to the kernel's storage dtype; biases stay fp32 (the GEMM epilogues
    add them in fp32)."""
    from paper_2105_04779_b200.attention import round_to_dtype

    f = lambda a: round_to_dtype(a, dtype)  # noqa: E731
    g = lambda a: np.asarray(a, np.float32).astype(np.float64)  # noqa: E731
    return O.Params(p.h, p.d_m, p.d_k, f(p.Wq), f(p.Wk), f(p.Wv), f(p.Wo), g(p.bq), g(p.bk), g(p.bv),
                    g(p.bo), p.include_key_bias, p.include_value_bias)
