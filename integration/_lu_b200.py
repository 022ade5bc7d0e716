"""rlra/_lu_b200.py -- the B200 backend of the reference's LU kernel seam.

Drop this file into the reference package next to ``_lu_cython`` and let
``rlra/backend.py`` accept ``RLRA_BACKEND=b200`` (integration/install_backend.py
does both on a copy of an installed reference).  Every ``kernels.plu`` call of
the reference (rlra/kernels.py:49) then runs the bit-exact GEPP of
librlra_b200.so on the GPU through its C ABI:

    int rlra_b200_plu_inplace(double* lu, int64_t m, int64_t n, int64_t* piv);

Contract = the Cython kernel's (rlra/_lu_cython.pyx:14): ``lu`` host
F-contiguous float64 m x n, overwritten with packed L\\U; ``piv`` host int64[m]
preloaded with 0..m-1, permuted in place; bit-identical results.
"""

import ctypes
import os

import numpy as np

_LIB = os.environ.get("RLRA_B200_LIB", "librlra_b200.so")
_lib = ctypes.CDLL(_LIB)
_lib.rlra_b200_plu_inplace.restype = ctypes.c_int
_lib.rlra_b200_plu_inplace.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
_lib.rlra_b200_last_error.restype = ctypes.c_char_p


def plu_inplace(lu, piv):
    """In-place packed LU with row pivoting (rlra/_lu_cython.pyx:14-55 contract)."""
    if not (isinstance(lu, np.ndarray) and lu.dtype == np.float64 and lu.ndim == 2 and lu.flags.f_contiguous):
        raise ValueError("Buffer dtype mismatch or not F-contiguous: lu must be a float64 Fortran-ordered matrix")
    if not (isinstance(piv, np.ndarray) and piv.dtype == np.int64 and piv.ndim == 1 and piv.flags.c_contiguous):
        raise ValueError("Buffer dtype mismatch: piv must be a contiguous int64 vector")
    m, n = lu.shape
    if piv.shape[0] < m:
        raise ValueError("piv shorter than the number of rows")
    if m == 0 or n == 0:
        return
    if not lu.flags.writeable or not piv.flags.writeable:
        raise ValueError("buffer source array is read-only")
    if _lib.rlra_b200_plu_inplace(lu.ctypes.data, m, n, piv.ctypes.data) != 0:
        raise RuntimeError(_lib.rlra_b200_last_error().decode(errors="replace"))
