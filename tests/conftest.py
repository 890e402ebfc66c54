import os
import sys

# the OpenMP oracle shares torch's libgomp in these processes; with libgomp's default
# active wait its threads contend with torch's pool (10x slower).  Read at libgomp init,
# so it is set before anything imports torch.
os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")

import pytest  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the CUDA extension")
    config.addinivalue_line("markers", "slow: long-running (full-size) case")


def pytest_collection_modifyitems(config, items):
    # GPU tests must run against the CUDA path; if no GPU is visible they are skipped
    # only when the caller selected them without a GPU (e.g. a CPU box running -m gpu).
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device visible")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
