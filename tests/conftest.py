import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
for p in (str(ROOT), str(ROOT / "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")


def _cuda_ok():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    # GPU tests are selected with -m gpu; on a box without a GPU they fail loudly
    # (no silent skip), except when the user deselects them with -m "not gpu".
    pass


@pytest.fixture(scope="session")
def gpu():
    if not _cuda_ok():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2105_04779_b200 as E

    E.capi.lib()  # raises ElattnUnavailable when the .so is missing: no fallback
    return E
