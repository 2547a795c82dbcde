import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "hefit_golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running oracle case")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


def cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def import_reference():
    """The unmodified reference package (hefit): the driver's offline install
    under baseline/_ref travels with the repo; /root/reference exists only in
    the build container.  None when neither is present."""
    import importlib
    for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "hefit")):
            if p not in sys.path:
                sys.path.append(p)
            try:
                return importlib.import_module("hefit")
            except Exception:
                return None
    return None


@pytest.fixture(scope="session")
def hefit():
    mod = import_reference()
    if mod is None:
        pytest.skip("reference package hefit not importable (baseline/_ref absent)")
    return mod


@pytest.fixture(autouse=True)
def _release_contexts():
    """A context owns a multi-GB device pool (keys, reserved working set) that
    is released when the object is destroyed; contexts caught in reference
    cycles (ciphertexts, closures of the threaded shard tests) would wait for
    the cyclic collector, and a long GPU session could pile them up to the
    180 GB of the device.  Collect after every test."""
    yield
    import gc
    gc.collect()
