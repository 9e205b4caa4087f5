"""The C ABI library builds for sm_100a, loads, and exports exactly what
include/genoiht_cuda.h declares; without a GPU the product fails loudly."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT, has_gpu

HEADER = os.path.join(ROOT, "include", "genoiht_cuda.h")
LIB = os.path.join(ROOT, "paper_1608_01398_b200", "libgenoiht_cuda.so")


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gi_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_1608_01398_b200", "csrc")],
                       check=True)
    return ctypes.CDLL(LIB)


def test_every_declared_symbol_is_exported(lib):
    names = _declared()
    assert len(names) >= 30
    for name in names:
        assert hasattr(lib, name), name


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_binding_covers_header():
    from paper_1608_01398_b200 import _native
    src = open(_native.__file__).read()
    for name in _declared():
        assert f'"{name}"' in src, name


def test_runtime_calls_without_gpu(lib):
    lib.gi_version.restype = ctypes.c_int
    assert lib.gi_version() == 100
    count = ctypes.c_int(-1)
    assert lib.gi_device_count(ctypes.byref(count)) == 0
    assert count.value >= 0
    lib.gi_red_partials.restype = ctypes.c_int64
    assert lib.gi_red_partials() > 0
    lib.gi_topk_slots.restype = ctypes.c_int64
    lib.gi_topk_slots.argtypes = [ctypes.c_int64, ctypes.c_int64]
    assert lib.gi_topk_slots(10000, 20) == 3 * 20


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    import paper_1608_01398_b200 as gi
    from paper_1608_01398_b200._native import NativeError
    with pytest.raises(NativeError, match="no CPU fallback|no CUDA device"):
        gi.PackedGenotypeMatrix.from_codes(np.zeros((8, 3), np.uint8))
