"""ctypes binding of librlra_b200.so (the C ABI in include/rlra_b200.h).

The product path has no CPU fallback: if the shared library is missing or no
CUDA device is visible, every operation raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes
import os
import re

from .errors import DeviceError, NativeUnavailable

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RLRA_B200_LIB") or os.path.join(_HERE, "_lib", "librlra_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "rlra_b200.h")

_c_i64 = ctypes.c_int64
_c_p = ctypes.c_void_p
_c_d = ctypes.c_double
_c_sz = ctypes.c_size_t
_c_i = ctypes.c_int

# name -> (restype, argtypes); mirrors include/rlra_b200.h
SIGNATURES = {
    "rlra_b200_abi_version": (_c_i, []),
    "rlra_b200_last_error": (ctypes.c_char_p, []),
    "rlra_b200_device_count": (_c_i, [_c_p]),
    "rlra_b200_launch_count": (ctypes.c_longlong, []),
    "rlra_b200_ktimer_enable": (_c_i, [_c_i]),
    "rlra_b200_ktimer_read": (_c_i, [ctypes.c_char_p, _c_p, _c_p]),
    "rlra_b200_plu_inplace": (_c_i, [_c_p, _c_i64, _c_i64, _c_p]),
    "rlra_b200_getrf_workspace": (_c_sz, [_c_i64, _c_i64]),
    "rlra_b200_getrf": (_c_i, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_sz, _c_p]),
    "rlra_b200_iota": (_c_i, [_c_p, _c_i64, _c_p]),
    "rlra_b200_getrf_block": (_c_i, [_c_p, _c_i64, _c_i64, _c_i64, _c_i, _c_p, _c_p, _c_p, _c_p, _c_p, _c_sz,
                                     _c_p]),
    "rlra_b200_lu_trsm_rows": (_c_i, [_c_p, _c_i64, _c_i64, _c_i, _c_i64, _c_i64, _c_p, _c_p]),
    "rlra_b200_lu_update_split": (_c_i, [_c_p, _c_i64, _c_p, _c_i64, _c_i64, _c_i, _c_i64, _c_i64, _c_i64, _c_i64,
                                         _c_p, _c_p]),
    "rlra_b200_count_nonzero_diag": (_c_i, [_c_p, _c_i64, _c_i64, _c_p, _c_p]),
    "rlra_b200_lu_basis": (_c_i, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_i64, _c_p]),
    "rlra_b200_lu_extract": (_c_i, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_i64, _c_p]),
    "rlra_b200_gemm_workspace": (_c_sz, [_c_i64, _c_i64, _c_i64]),
    "rlra_b200_dgemm": (_c_i, [_c_i, _c_i, _c_i64, _c_i64, _c_i64, _c_d, _c_p, _c_i64, _c_p, _c_i64,
                               _c_d, _c_p, _c_i64, _c_p, _c_sz, _c_p]),
    "rlra_b200_oz_prep_workspace": (_c_sz, [_c_i64, _c_i64, _c_i]),
    "rlra_b200_oz_prep": (_c_i, [_c_p, _c_i64, _c_i64, _c_i64, _c_i, _c_p, _c_sz, _c_p]),
    "rlra_b200_oz_gemm_workspace": (_c_sz, [_c_i, _c_i64, _c_i64, _c_i64, _c_i]),
    "rlra_b200_oz_gemm": (_c_i, [_c_i, _c_p, _c_i64, _c_i64, _c_i, _c_p, _c_i64, _c_i64, _c_p, _c_i64,
                                 _c_p, _c_sz, _c_p]),
    "rlra_b200_oz_scale_workspace": (_c_sz, [_c_i64, _c_i64]),
    "rlra_b200_oz_scale": (_c_i, [_c_p, _c_i64, _c_i64, _c_i64, _c_i, _c_p, _c_p, _c_sz, _c_p]),
    "rlra_b200_oz_prep_ex": (_c_i, [_c_p, _c_i64, _c_i64, _c_i64, _c_i, _c_p, _c_p, _c_sz, _c_p]),
    "rlra_b200_oz_cols_pad": (_c_i64, [_c_i64]),
    "rlra_b200_oz_norms": (_c_i, [_c_p, _c_i64, _c_i64, _c_i64, _c_i, _c_p, _c_sz, _c_p]),
    "rlra_b200_oz_guard_limit": (_c_d, [_c_i64]),
    "rlra_b200_oz_guard": (_c_i, [_c_p, _c_i64, _c_i64, _c_p, _c_p]),
    "rlra_b200_oz_norms_cols": (_c_i, [_c_p, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_i, _c_p, _c_sz, _c_p]),
    "rlra_b200_oz_scale_provisional": (_c_i, [_c_i64, _c_i64, _c_i64, _c_i, _c_p, _c_sz, _c_p]),
    "rlra_b200_oz_residue_cols": (_c_i, [_c_p, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_i, _c_p, _c_sz, _c_p]),
    "rlra_b200_oz_norms_finish": (_c_i, [_c_p, _c_i64, _c_i64, _c_i64, _c_i, _c_p, _c_sz, _c_p, _c_p]),
    "rlra_b200_oz_bscale": (_c_i, [_c_p, _c_i64, _c_i64, _c_i64, _c_i, _c_p, _c_p]),
    "rlra_b200_oz_gemm_ex": (_c_i, [_c_i, _c_p, _c_i64, _c_i64, _c_i, _c_p, _c_i64, _c_i64, _c_p, _c_i64,
                                    _c_p, _c_sz, _c_p, _c_i, _c_p]),
    "rlra_b200_oz_colsq": (_c_i, [_c_i, _c_i64, _c_i64, _c_i, _c_i64, _c_p, _c_sz, _c_p, _c_i, _c_p]),
    "rlra_b200_geqrf_workspace": (_c_sz, [_c_i64, _c_i64]),
    "rlra_b200_geqrf": (_c_i, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_sz, _c_p]),
    "rlra_b200_orgqr": (_c_i, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_sz, _c_p]),
    "rlra_b200_chol_inv_max_l": (_c_i, []),
    "rlra_b200_chol_shift_diag": (_c_i, [_c_p, _c_i64, _c_i64, _c_d, _c_p]),
    "rlra_b200_diag_ratio_flag": (_c_i, [_c_p, _c_i64, _c_i64, _c_d, _c_p, _c_p]),
    "rlra_b200_gram_identity_flag": (_c_i, [_c_p, _c_i64, _c_i64, _c_d, _c_p, _c_p]),
    "rlra_b200_chol_inv": (_c_i, [_c_p, _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_d, _c_p]),
    "rlra_b200_trsm_workspace": (_c_sz, [_c_i64, _c_i64]),
    "rlra_b200_trsm_rt": (_c_i, [_c_p, _c_i64, _c_i64, _c_p, _c_i64, _c_i64, _c_p, _c_sz, _c_p]),
    "rlra_b200_trsm_un": (_c_i, [_c_p, _c_i64, _c_i64, _c_p, _c_i64, _c_i64, _c_p, _c_sz, _c_p]),
    "rlra_b200_apply_inv_row_perm": (_c_i, [_c_p, _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_p, _c_i64, _c_p]),
    "rlra_b200_resid_sumsq_block": (_c_i, [_c_p, _c_i64, _c_i64, _c_p, _c_p, _c_i64, _c_p, _c_i64, _c_p, _c_p]),
    "rlra_b200_dd_finish": (_c_i, [_c_p, _c_i64, _c_p, _c_p]),
    "rlra_b200_spmm_csr": (_c_i, [_c_p, _c_p, _c_p, _c_i64, _c_p, _c_i64, _c_i64, _c_p, _c_i64, _c_p]),
    "rlra_b200_svd_jacobi_max_l": (_c_i, []),
    "rlra_b200_svd_jacobi_workspace": (_c_sz, [_c_i64, _c_i64]),
    "rlra_b200_svd_jacobi": (_c_i, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_p, _c_i64, _c_p, _c_p,
                                    _c_sz, _c_p]),
    "rlra_b200_diag_absmin": (_c_i, [_c_p, _c_i64, _c_i64, _c_p, _c_p]),
    "rlra_b200_sumsq_workspace": (_c_sz, [_c_i64, _c_i64]),
    "rlra_b200_sumsq": (_c_i, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_sz, _c_p]),
    "rlra_b200_colsumsq": (_c_i, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p]),
    "rlra_b200_transpose": (_c_i, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_i64, _c_p]),
    "rlra_b200_normal_workspace": (_c_sz, [_c_i64]),
    "rlra_b200_normal_stream_words": (_c_i64, [_c_i64]),
    "rlra_b200_normal_tail_cap": (_c_i64, [_c_i64]),
    "rlra_b200_normal_begin": (_c_i, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                      _c_i64, _c_p, _c_p, _c_p, _c_p, _c_sz, _c_p]),
    "rlra_b200_normal_views": (_c_i, [_c_i64, _c_p, _c_p, _c_p, _c_p]),
    "rlra_b200_normal_finish": (_c_i, [_c_i64, _c_p, _c_p, _c_p, _c_i64, _c_p, _c_p, _c_p, _c_sz, _c_p]),
}

_lib = None


def header_symbols(path=HEADER_PATH):
    """Every function the public header declares (used by the ABI tests)."""
    with open(path) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(rlra_b200_[a-z0-9_]+)\s*\(", text)))


def load():
    """Load the shared library (no GPU needed); raise loudly when missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeUnavailable(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.rlra_b200_abi_version() != 1:
        raise NativeUnavailable("librlra_b200.so ABI version mismatch")
    _lib = lib
    return lib


def call(name, *args):
    """Invoke a status-returning entry point; map failures to DeviceError."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.rlra_b200_last_error().decode(errors="replace")
        raise DeviceError(f"{name} failed ({rc}): {msg}")
    return rc


def query(name, *args):
    """Invoke a size query (returns size_t)."""
    return int(getattr(load(), name)(*args))
