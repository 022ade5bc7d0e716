"""The native-kernel seam: drop-in for the reference's backend.plu_inplace
(rlra/backend.py:32 -> rlra/_lu_cython.pyx:14-55).

``plu_inplace(lu, piv)`` takes the same caller-owned host buffers (F-contiguous
float64 m x n, int64[m] preloaded with 0..m-1), factors on the B200 through the
C ABI ``rlra_b200_plu_inplace`` and writes back bit-identical results.
"""

from __future__ import annotations

import numpy as np

from . import _native

BACKEND = "b200"


def plu_inplace(lu, piv):
    if not (isinstance(lu, np.ndarray) and lu.dtype == np.float64 and lu.ndim == 2
            and lu.flags.f_contiguous and lu.flags.writeable):
        raise ValueError("lu must be a writeable F-contiguous float64 2-d array")
    if not (isinstance(piv, np.ndarray) and piv.dtype == np.int64 and piv.ndim == 1
            and piv.shape[0] == lu.shape[0] and piv.flags.c_contiguous):
        raise ValueError("piv must be a contiguous int64 array of length m")
    m, n = lu.shape
    _native.call("rlra_b200_plu_inplace", lu.ctypes.data, m, n, piv.ctypes.data)
