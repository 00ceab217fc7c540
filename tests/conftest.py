import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: oracle convergence studies (tens of seconds)")


def cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if cuda_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


def pytest_sessionfinish(session, exitstatus):
    """Write the per-field parity metric of every GPU parity test (BASELINE.md
    §2) next to the run's other GPU evidence when gpurun_out/ exists."""
    try:
        import json
        from tests import test_gpu_parity as tp   # noqa: F401
    except Exception:
        try:
            import json
            import test_gpu_parity as tp          # noqa: F401
        except Exception:
            return
    out = os.path.join(ROOT, "gpurun_out")
    if tp.PER_FIELD and os.path.isdir(out):
        with open(os.path.join(out, "parity_per_field.json"), "w") as fh:
            json.dump(tp.PER_FIELD, fh, indent=1)
