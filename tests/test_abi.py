"""The C-ABI shared library loads and exports every symbol include/rlra_b200.h
declares; the Python bindings cover exactly that set; without a GPU the
product path fails loudly (no CPU fallback).  CPU only."""

import ctypes
import subprocess

import numpy as np
import pytest

from paper_2002_07138_b200 import _native


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    syms = _native.header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/rlra_b200.h but not exported"


def test_bindings_match_header():
    assert sorted(_native.SIGNATURES) == _native.header_symbols()


def test_only_abi_symbols_are_exported():
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True)
    exported = sorted({l.split()[-1] for l in out.stdout.splitlines() if " T " in l})
    assert exported == _native.header_symbols()


def test_abi_version_and_error_string():
    lib = _native.load()
    assert lib.rlra_b200_abi_version() == 1
    assert isinstance(lib.rlra_b200_last_error(), bytes)


def test_workspace_queries_need_no_gpu():
    lib = _native.load()
    assert lib.rlra_b200_getrf_workspace(20000, 220) > 0
    assert lib.rlra_b200_geqrf_workspace(10000, 220) > 0


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    import paper_2002_07138_b200 as P

    with pytest.raises(P.NativeUnavailable):
        P.powerlu(np.eye(20), 3, q_os=1, v=3, seed=0)
    with pytest.raises(P.DeviceError):
        lu = np.asfortranarray(np.eye(4))
        P.plu_inplace(lu, np.arange(4, dtype=np.int64))
