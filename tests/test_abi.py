"""The C-ABI library loads and exports every symbol include/dade.h declares (no GPU needed)."""
import ctypes as C
import os
import re

import pytest

from paper_2404_16322_b200 import dade

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "dade.h")).read()
    return sorted(set(re.findall(r"\b(dade_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    from paper_2404_16322_b200 import build
    build.build()
    return dade.lib()


def test_header_declares_the_boundary():
    names = declared_symbols()
    for req in ("dade_fit_rotation", "dade_calibrate", "dade_build_ivf", "dade_search", "dade_merge_topk"):
        assert req in names


def test_every_declared_symbol_is_exported(L):
    for name in declared_symbols():
        assert hasattr(L, name), name
    assert set(dade._SIGS) | {"dade_last_error"} >= set(declared_symbols())


def test_argument_errors_before_touching_cuda(L):
    h = C.c_void_p()
    assert L.dade_create(0, None, 0, C.byref(h)) == 1      # ERR_ARG: D <= 0
    assert b"positive" in L.dade_last_error()
    assert L.dade_create(0, None, 100, C.byref(h)) == 8    # ERR_UNSUPPORTED: D % 16
    assert L.dade_destroy(None) == 0


def test_no_gpu_fails_loudly(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    st = L.dade_create(0, None, 128, C.byref(h))
    assert st == 6  # ERR_CUDA: no device -> loud error, never a CPU fallback
