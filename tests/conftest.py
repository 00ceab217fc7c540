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
    """Write the parity numbers of the GPU tests (per-field metric of every parity
    test; K and worst sampled error of every full-size golden case)
    next to the run's other GPU evidence when gpurun_out/ exists."""
    import importlib
    import json
    out = os.path.join(ROOT, "gpurun_out")
    if not os.path.isdir(out):
        return
    for mod, attr, fname in (("test_gpu_parity", "PER_FIELD", "parity_per_field.json"),
                             ("test_gpu_fullsize", "RESULTS", "fullsize_parity.json")):
        m = sys.modules.get(mod) or sys.modules.get("tests." + mod)
        if m is None:
            continue
        data = getattr(m, attr, None)
        if data:
            with open(os.path.join(out, fname), "w") as fh:
                json.dump(data, fh, indent=1)
