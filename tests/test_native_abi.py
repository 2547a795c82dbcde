"""CPU checks of the C-ABI boundary: the library builds for sm_100a, loads
without a GPU, and exports every function include/hc.h declares with the
signature table the Python binding uses."""

import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hc.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hc_[a-z0-9_]+)\s*\(", src)) - {"hc_reduce_fn"})


@pytest.fixture(scope="module")
def lib():
    from paper_2403_14111_b200 import _native
    _native.build()
    return _native.lib()


def test_header_symbols_exported(lib):
    from paper_2403_14111_b200 import _native
    names = declared()
    assert len(names) >= 35
    out = subprocess.check_output(["nm", "-D", "--defined-only", _native.LIB_PATH]).decode()
    exported = set(re.findall(r" T (hc_[a-z0-9_]+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    assert set(names) == set(_native.SIGNATURES)
    for n in names:
        assert getattr(lib, n) is not None


def test_library_is_sm100a():
    from paper_2403_14111_b200 import _native
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH]).decode()
    assert "sm_100a" in out


def test_no_gpu_compute_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2403_14111_b200 as P
    with pytest.raises(RuntimeError):
        P.CKKSContext("tiny", 16)
