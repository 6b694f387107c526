"""The reference's own attention tests, re-pointed at the C++ drop-in
(include/elattn_gpu.hpp) and run on the GPU (tests/cpp/test_gpu_attention.cpp)."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parent / "cpp" / "test_gpu_attention"


@pytest.mark.gpu
def test_cpp_dropin_against_reference(gpu):
    if not BIN.exists():
        pytest.skip("tests/cpp/test_gpu_attention not built (needs /root/reference headers at build time)")
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
