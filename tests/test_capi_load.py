"""CPU-side checks of the C-ABI library and the host logic (no compute calls)."""
import ctypes
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

import paper_2105_04779_b200 as E
from paper_2105_04779_b200 import capi
from paper_2105_04779_b200.attention import DTYPE_BF16, DTYPE_F32, round_to_dtype

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "elattn_gpu.h").read_text()
    return sorted(set(re.findall(r"\b(elattn_gpu_[a-z_]+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    L = capi.lib()
    declared = header_symbols()
    assert declared, "no symbols parsed from include/elattn_gpu.h"
    for name in declared:
        assert hasattr(L, name), name
    assert set(declared) == set(capi.EXPORTED_SYMBOLS)
    nm = subprocess.run(["nm", "-D", "--defined-only", str(capi.LIB_PATH)], capture_output=True, text=True).stdout
    for name in declared:
        assert re.search(rf"\bT {name}\b", nm), name
    assert "sm_100a" in E.version()


def test_library_is_sm100a_native():
    out = subprocess.run(["cuobjdump", "--list-elf", str(capi.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", str(capi.LIB_PATH)], capture_output=True, text=True).stdout
    # Blackwell-native evidence: tcgen05.mma (UTCHMMA), TMA (UTMALDG), TMEM ld/st (LDTM/STTM)
    for op in ("UTCHMMA", "UTMALDG", "LDTM", "STTM"):
        assert re.search(rf"\b{op}\b", sass), op
    # and no legacy mma.sync / Hopper wgmma tensor paths
    assert not re.search(r"(?<!UTC)\bHMMA\b", sass) and "HGMMA" not in sass


def test_errors_without_device_are_statuses_not_crashes():
    L = capi.lib()
    h = ctypes.c_void_p()
    arr = np.zeros(64)
    rc = L.elattn_gpu_params_create(0, 8, 4, 0, 1, 1, *([arr.ctypes.data] * 8), ctypes.byref(h))
    assert rc == capi.ERR_PARAM
    assert b"h, d_m, d_k" in L.elattn_gpu_last_error_message()
    with pytest.raises(E.ParamError):
        capi.check(rc)
    rc = L.elattn_gpu_params_create(1, 8, 4, 7, 1, 1, *([arr.ctypes.data] * 8), ctypes.byref(h))
    assert rc == capi.ERR_PARAM
    # null handle on compute entry points is a PARAM error, not a segfault
    assert L.elattn_gpu_el_attention_step(None, None, None, None, 1, 1, 1, None, None, 0, None) == capi.ERR_PARAM
    assert L.elattn_gpu_workspace_size(None, 1, 1, 1) == 0


def test_round_to_dtype_is_rne():
    x = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -2.5, 0.0, 3.0e38, 1e-40])
    got = round_to_dtype(x, DTYPE_BF16)
    import torch

    want = torch.tensor(x, dtype=torch.float64).to(torch.float32).to(torch.bfloat16).double().numpy()
    assert np.array_equal(got, want)
    assert np.array_equal(round_to_dtype(x, DTYPE_F32), x.astype(np.float32).astype(np.float64))


def test_fold_layout_matches_reference_convention():
    # fold_el_queries (attention.hpp:293-304): row = b*h + i
    h, d_m = 3, 5
    qs = [E.ElQuery(np.arange(h * d_m, dtype=float).reshape(h, d_m) + 100 * b, np.arange(h) + 10 * b)
          for b in range(4)]
    q, s = E.fold_el_queries(qs, h, d_m)
    for b in range(4):
        for i in range(h):
            assert np.array_equal(q[b * h + i], qs[b].elq[i]) and s[b * h + i] == qs[b].s[i]
