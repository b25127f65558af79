import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def has_cuda() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)
        return cache[name]
    return load


@pytest.fixture(scope="session", autouse=True)
def _built_oracle():
    from oracle import oracle
    oracle.lib()


def reference_convkit():
    """The reference package (baseline/_ref, else /root/reference in the build
    container) for side-by-side interface checks; None where it is absent."""
    import importlib
    import tempfile
    for path in (os.path.join(ROOT, "baseline", "_ref"),
                 os.path.join("/root", "reference", "pkg", "src")):
        if os.path.isdir(os.path.join(path, "convkit")):
            if path not in sys.path:
                sys.path.append(path)
            os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="ck_numba_"))
            try:
                return importlib.import_module("convkit")
            except Exception:
                return None
    return None
