import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
# The unmodified reference package, when installed into baseline/_ref (see
# tests/test_gpu_dropin_reference.py): importable by the whole session, so the
# drop-in modules bind the reference's exception classes at import, as in a
# reference run with the device path patched in (errors.py).
_REF = os.path.join(ROOT, "baseline", "_ref")
if os.path.isdir(os.path.join(_REF, "iscsim")) and _REF not in sys.path:
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join("/tmp", "numba_cache_iscsim_tests"))
    sys.path.append(_REF)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
