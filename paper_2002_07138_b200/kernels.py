"""Device versions of the reference's dense factorization kernels
(rlra/kernels.py:20-117): pivoted LU, economy QR, pseudoinverse solve.
All arithmetic runs in librlra_b200.so; nothing here computes on the host.
"""

from __future__ import annotations

import os
from typing import NamedTuple

import torch

from . import ops
from .errors import IllPosedPseudoinverse

PINV_RTOL = 1e-12  # rlra/kernels.py:17


class PivotedLU(NamedTuple):
    L: torch.Tensor  # m x r unit-lower
    U: torch.Tensor  # r x n upper
    p: torch.Tensor  # row permutation: A[p, :] = L @ U
    nonzero_diag: torch.Tensor  # device int64[1]: count_nonzero(diag(U))


def plu_(a, want_l=True, want_u=True):
    """kernels.plu (rlra/kernels.py:37-54) on a device matrix, factoring `a` IN
    PLACE (callers pass a scratch copy when they still need the input)."""
    piv, cnt = ops.getrf_(a)
    l, u = ops.lu_extract(a, want_l, want_u)
    return PivotedLU(l, u, piv, cnt)


def plu(a):
    """Non-destructive kernels.plu."""
    return plu_(_copy(a))


def _copy(a):
    out = ops.fmat(a.shape[0], a.shape[1], a.device)
    out.copy_(a)
    return out


def eqr_(a):
    """kernels.eqr (rlra/kernels.py:57-61), destroying `a`: returns (Q, QR)."""
    qr = ops.QR(a)
    return qr.q(), qr


class _CholFactor:
    """QR factor from CholeskyQR (pinv_factor_): q() and r_view() like ops.QR."""

    def __init__(self, q, r):
        self._q, self._r = q, r

    def q(self):
        return self._q

    def r_view(self):
        return self._r


PINV_QR = os.environ.get("RLRA_B200_PINV_QR", "chol")
PINV_CHOL_MARGIN = 1e4  # CholeskyQR's R is trusted for the rank test only this far above PINV_RTOL


def pinv_factor_(l):
    """kernels.pinv_factor (rlra/kernels.py:64-79) on a scratch copy of `l`.

    Raises IllPosedPseudoinverse when min |R_ii| <= PINV_RTOL * ||L||_F."""
    m, n = l.shape
    if m < n:
        raise ValueError(f"need a tall matrix, got {(m, n)}")
    fro2 = ops.sumsq(l)
    if PINV_QR == "chol" and n > 0:
        # CholeskyQR2 / shifted CholeskyQR3 (tall products on the int8 engine)
        # instead of the latency-bound Householder panels (C4: G 50000 x 720).
        # R = Q^T L; the reference's rank test on its diagonal is decided here
        # only when min |R_ii| clears the threshold by PINV_CHOL_MARGIN (Cholesky
        # R is accurate to ~u cond); otherwise -- or when the Cholesky declined
        # -- the Householder path below decides exactly as rlra/kernels.py:64-79.
        # CholeskyQR2 first (two steps, cond(L) up to ~1e7 -- C4's G), shifted
        # CholeskyQR3 when it declines (cond up to ~u^-1), then Householder
        for method in (ops.cholqr2, ops.scholqr3):
            q, flag = method(l)
            _, r = ops.lu_extract(ops.tn_tall(q, l), want_l=False)
            dmin = ops.diag_absmin(r)
            vals = torch.cat([dmin, fro2, flag.to(torch.float64)]).cpu()
            if not int(vals[2]):
                if float(vals[0]) > PINV_CHOL_MARGIN * PINV_RTOL * float(vals[1]) ** 0.5:
                    return _CholFactor(q, r)
                break  # near the rank threshold: Householder decides, as the reference does
    work = _copy(l)
    qr = ops.QR(work)
    dmin = ops.diag_absmin(qr.r_view())
    vals = torch.cat([dmin, fro2]).cpu()
    if float(vals[0]) <= PINV_RTOL * float(vals[1]) ** 0.5:
        raise IllPosedPseudoinverse(f"matrix of shape {(m, n)} is numerically rank-deficient")
    return qr


def pinv_transpose_apply(l, m_):
    """(L^T)^+ M = Q R^{-T} M (rlra/kernels.py:92-96)."""
    qr = pinv_factor_(l)
    q = qr.q()
    prep = ops.tall_prep(q, m_.shape[1])  # Q's residues while the triangular solve runs
    x = _copy(m_)
    ops.trsm_rt_(qr.r_view(), x)
    return ops.tall_times(q, x, prep)
