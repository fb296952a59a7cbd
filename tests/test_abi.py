"""-m "not gpu": the C-ABI library loads and exports every symbol include/fl_attn.h
declares; host-only logic (shard ranges, validation that returns before any
CUDA call) behaves as documented.  No compute calls here."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "fl_attn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fl_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    from paper_2511_02043_b200 import _lib
    if not os.path.exists(_lib.SO_PATH):
        from paper_2511_02043_b200 import build
        build.build()
    return _lib.lib()


def test_exports_every_declared_symbol(L):
    names = header_functions()
    assert len(names) >= 10, names
    from paper_2511_02043_b200 import _lib
    assert set(names) == set(_lib.EXPORTS), (set(names) ^ set(_lib.EXPORTS))
    for n in names:
        assert hasattr(L, n), n


def test_abi_version_and_status_strings(L):
    from paper_2511_02043_b200 import _lib
    assert L.fl_abi_version() == _lib.ABI_VERSION == 4
    assert L.fl_status_string(0) == b"FL_OK"
    assert L.fl_status_string(2) == b"FL_ERR_UNSUPPORTED"


def test_validation_before_any_cuda_call(L):
    from paper_2511_02043_b200 import _lib
    assert L.fl_attn_fwd(None) == 1
    a = _lib.AttnArgs()
    a.var.abi_version = 99
    assert L.fl_attn_fwd(C.byref(a)) == 7          # FL_ERR_ABI_VERSION
    a.var.abi_version = _lib.ABI_VERSION
    assert L.fl_attn_fwd(C.byref(a)) == 1          # q/k/v/o missing
    assert b"required" in L.fl_last_error()


@pytest.mark.parametrize("units,world", [(128, 1), (128, 8), (7, 3), (3, 8), (512, 6), (0, 4)])
def test_shard_range_partitions(L, units, world):
    from paper_2511_02043_b200 import fl
    spans = [fl.shard_range(units, world, r) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == units
    for (b0, e0), (b1, e1) in zip(spans, spans[1:]):
        assert e0 == b1
    sizes = [e - b for b, e in spans]
    assert max(sizes) - min(sizes) <= 1
