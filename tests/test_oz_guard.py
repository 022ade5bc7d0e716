"""Dynamic-range guard of the emulated pass products (rlra_b200_oz_guard,
host-only: no GPU needed).

The int8 engine scales all of A by ONE power of two, so its error is
normwise in N_A = max row/column norm (csrc/ozaki.cu accuracy note):
    |err_ij| <= 2^-54 sqrt(K) N_A ||B_j|| + 2^-53 sqrt(K) ||A_i|| ||B_j|| + 2^-52 ||A_i|| ||B_j||.
The guard admits an orientation only when N_A / min_i ||A_i|| <= T(K) =
2 (K-2)/sqrt(K) - 2, which makes that bound <= K 2^-53 ||A_i|| ||B_j|| (the
classical DGEMM bound); everything else goes to the DMMA GEMM.
"""

import math
import struct

import numpy as np
import pytest

from paper_2002_07138_b200 import ops


def header(max_ss, min_row_ss, min_col_ss, nonfinite=0, e_a=0, nonint=1):
    bits = lambda x: struct.unpack("<Q", struct.pack("<d", x))[0] if x is not None else 0xFFFFFFFFFFFFFFFF  # noqa: E731
    raw = struct.pack("<iiQQQII", e_a, 0, bits(max_ss), bits(min_row_ss), bits(min_col_ss), nonfinite, nonint)
    return raw + b"\0" * (ops.OZ_HEADER_BYTES - len(raw))


def limit(k):
    from paper_2002_07138_b200 import _native

    return _native.load().rlra_b200_oz_guard_limit(k)


def test_limit_formula_and_bound():
    for k in (5, 100, 2000, 10000, 20000, 133120):
        t = limit(k)
        assert t == pytest.approx(2 * (k - 2) / math.sqrt(k) - 2)
        # the guard's promise: 2^-54 sqrt(K) T + 2^-53 sqrt(K) + 2^-52 <= K 2^-53
        assert 2.0 ** -54 * math.sqrt(k) * t + 2.0 ** -53 * math.sqrt(k) + 2.0 ** -52 <= k * 2.0 ** -53 * (1 + 1e-12)
    assert limit(4) == 0.0 and limit(1) == 0.0


def test_guard_decisions():
    m, n = 20000, 10000
    tn, tt = limit(n), limit(m)
    # balanced A (the C1-C5 shapes): both orientations on the int8 engine
    assert ops.oz_guard(header(4.0, 1.0, 1.0), m, n) == (True, True)
    # rows graded just inside / outside T(n): only NN decides on rows
    assert ops.oz_guard(header((0.99 * tn) ** 2, 1.0, (0.99 * tn) ** 2), m, n) == (True, True)
    assert ops.oz_guard(header((1.01 * tn) ** 2, 1.0, (1.01 * tn) ** 2), m, n) == (False, True)
    # columns graded beyond T(m): TN only
    assert ops.oz_guard(header((1.01 * tt) ** 2, (1.01 * tt) ** 2, 1.0), m, n) == (True, False)
    # NaN / Inf anywhere: both to DMMA
    assert ops.oz_guard(header(4.0, 1.0, 1.0, nonfinite=1), m, n) == (False, False)
    # A = 0: exact either way
    assert ops.oz_guard(header(0.0, 0.0, 0.0), m, n) == (True, True)
    # a zero row (or squares that underflow) next to non-zero ones: rejected
    assert ops.oz_guard(header(1.0, 0.0, 1.0), m, n) == (False, True)
    assert ops.oz_guard(header(1.0, 1.0, 1e-320), m, n) == (True, False)
    # everything tiny (norms below 2^-480): the scale leaves the normal range
    assert ops.oz_guard(header(2.0 ** -970, 2.0 ** -970, 2.0 ** -970), m, n) == (False, False)
    # integer-valued A: DMMA (exact products would turn exact dependencies into exact zero pivots)
    assert ops.oz_guard(header(4.0, 1.0, 1.0, nonint=0), m, n) == (False, False)
    # tiny K: no admissible ratio
    assert ops.oz_guard(header(1.0, 1.0, 1.0), 4, 4) == (False, False)


def test_guard_on_the_benchmark_configs():
    """C2-C5 (BASELINE.json configs) stay on the int8 engine: their measured
    row/column norm ratios (factor form, noise included) are inside T(K)."""
    rho = {"C2": (125.3, 87.0, 20000, 10000), "C3": (2.1, 2.0, 16384, 16384), "C4": (40.3, 33.8, 50000, 50000),
           "C5": (7.9, 2.8, 262144, 32768)}
    for name, (rr, rc, m, n) in rho.items():
        assert ops.oz_guard(header(rr * rr, 1.0, (rr / rc) ** 2), m, n) == (True, True), name


def test_header_decoding():
    h = np.frombuffer(header(16.0, 4.0, None, 0), dtype=np.uint8)
    assert ops.oz_guard_stats(h) == (4.0, 2.0, float("inf"), False, False)
    assert ops.oz_guard_stats(np.frombuffer(header(1.0, 1.0, 1.0, nonint=0), np.uint8))[4] is True
