import os
import sys

import pytest

# Several EP ranks share one device in the concurrent GPU tests (gpu_util.
# run_concurrent), each on its own streams.  With the default 8 hardware
# connections, streams of different ranks can map onto one connection and be
# serialised behind each other (a rank's kernels queued behind a peer's kernel
# that waits for them).  32 connections keep every rank's streams independent.
# Must be set before the CUDA context exists.
os.environ["CUDA_DEVICE_MAX_CONNECTIONS"] = "32"

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no GPU in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "reference_vectors.json")) as f:
        return json.load(f)
