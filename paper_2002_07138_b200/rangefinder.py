"""Power-iteration row-space basis for any pass budget v >= 2 on device
(rlra/rangefinder.py:20-176, the paper's Alg. 7 generalised to any v).

Same control flow, Omega shapes and pass accounting as the reference: even v
draws Omega m x l and starts with A^T Omega, odd v draws Omega n x l; interior
renormalisations are the row-unpermuted L of a partial-pivot LU (bit-exact
GEPP, K3); the last step is a Householder QR (K4) -- or, for powerlu's
internal basis, CholeskyQR2 with the Householder QR as fallback.  The exact-zero-diagonal
RankCollapse checks (rlra/rangefinder.py:55-64) are evaluated on device and
raised when the basis is handed back, with the reference's attributes.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import NamedTuple

import torch

from . import core, ops
from .device import as_accessor
from .errors import RankCollapse


class RangeBasis(NamedTuple):
    V: torch.Tensor  # n x l, orthonormal columns (device)
    passes_used: int


class SketchLU(NamedTuple):
    """rlra/rangefinder.py:25-28 (device tensors)."""

    L: torch.Tensor  # m x l, unit-diagonal lower trapezoidal
    U: torch.Tensor  # l x l
    p: torch.Tensor  # row permutation of the sketch


@dataclass(frozen=True)
class PowerParams:
    """Sketch-size bookkeeping l = k + q_os, exponent p, passes v = 2p + 2
    (rlra/rangefinder.py:31-52; host-only arithmetic)."""

    l: int
    p: int
    v: int
    q_oversample: int

    @classmethod
    def from_power(cls, k, q_oversample, p):
        return cls(l=k + q_oversample, p=p, v=2 * p + 2, q_oversample=q_oversample)

    @classmethod
    def from_passes(cls, k, q_oversample, v):
        if v < 2 or v % 2:
            raise ValueError(f"pass budget {v} has no power-exponent equivalent")
        return cls(l=k + q_oversample, p=(v - 2) // 2, v=v, q_oversample=q_oversample)


class RankChecks:
    """Deferred _check_width calls: (device nonzero-count, requested) pairs,
    resolved with a single host sync in call order."""

    def __init__(self):
        self._items = []
        self._cholqr = None  # (flag, Z) of a deferred CholeskyQR2 basis
        self._resolved = []  # host values of the first len(_resolved) counts

    def add(self, count, requested):
        self._items.append((count, int(requested)))

    def defer_cholqr(self, flag, z):
        self._cholqr = (flag, z)

    def _fetch(self, extra=None):
        """Every unresolved count (and `extra`) in ONE device->host transfer."""
        pend = [c.view(-1) for c, _ in self._items[len(self._resolved):]]
        if extra is not None:
            pend.append(extra.view(-1).to(torch.int64))
        if not pend:
            return []
        dev_vals = torch.cat(pend) if len(pend) > 1 else pend[0]
        host = torch.empty(dev_vals.shape, dtype=dev_vals.dtype, pin_memory=dev_vals.is_cuda)
        host.copy_(dev_vals, non_blocking=True)  # pinned: no staging copy (r01 verdict: pageable fetch gap)
        if dev_vals.is_cuda:
            torch.cuda.current_stream(dev_vals.device).synchronize()
        vals = host.tolist()
        n = len(vals) - (extra is not None)
        self._resolved.extend(int(v) for v in vals[:n])
        return vals[n:]

    def cholqr_declined(self):
        """The parked CholeskyQR2 flag: None when no basis was deferred, else
        (declined, Z).  The counts queued so far come back in the same host
        round trip, so a call that does not decline syncs exactly once."""
        if self._cholqr is None:
            return None
        flag, z = self._cholqr
        self._cholqr = None
        return bool(int(self._fetch(flag)[0])), z

    def raise_if_collapsed(self):
        """Raise RankCollapse for the first count (in call order) below its
        requested width; only counts not yet resolved cost a transfer."""
        if not self._items:
            return
        self._fetch()
        items, counts = self._items, self._resolved
        self._items, self._resolved = [], []
        for achieved, (_, requested) in zip(counts, items):
            if achieved < requested:
                raise RankCollapse(int(achieved), requested)


def _validate(a, l, lower=1):
    """rlra/rangefinder.py:80-83."""
    m, n = a.shape
    if not lower <= l <= min(m, n):
        raise ValueError(f"sketch width l={l} outside {lower}..min{(m, n)}")


def qr_basis_(x, checks, method="householder"):
    """rlra/rangefinder.py:67-70 (destroys x, except on the CholeskyQR2 path).

    method="chol" (powerlu's internal basis): CholeskyQR2 -- same range as the
    Householder Q, columns possibly of opposite sign, which no powerlu output
    depends on.  Its decline flag (non-SPD Gram / condition bound) is NOT read
    here: the flag and x are parked in `checks` (checks.cholqr_declined(), one
    host sync at the end of the driver) and the caller redoes the basis on the
    Householder path if it was raised -- rank collapse keeps the reference's
    exception there.  method="householder_now": Householder unconditionally."""
    if method == "chol" and x.shape[0] >= x.shape[1] > 0:
        # CholeskyQR2 for l <= chol_inv_max_l (one-CTA Cholesky); wider sketches
        # (C3 l = 1024, C5 l = 544, whose cond(Z) reaches 1e9+) by shifted
        # CholeskyQR3 with blocked Choleskys -- Householder panels are latency
        # bound (one cluster exchange per column, 13-17 ms at those widths)
        if x.shape[1] <= ops.cholqr_max_l():
            q, flag = ops.cholqr2(x)
        else:
            q, flag = ops.scholqr3(x)
        checks.defer_cholqr(flag, x)
        return q
    qr = ops.QR(x)
    checks.add(ops.count_nonzero_diag(qr.r_view()), x.shape[1])
    return qr.q()


def lu_basis_(x, checks):
    """rlra/rangefinder.py:73-77: row-unpermuted L of lu(x) (destroys x)."""
    piv, cnt = ops.getrf_(x)
    checks.add(cnt, x.shape[1])
    return ops.lu_basis(x, piv)


def general_power_basis_v(a, l, v, seed, *, _checks=None, _qr="householder"):
    """rlra/rangefinder.py:144-176; consumes exactly v - 1 passes."""
    if getattr(a, "is_sharded", False):
        from .distributed import api_general_power_basis_v

        return api_general_power_basis_v(a, l, v, seed)
    a = as_accessor(a)
    _validate(a, l)
    if v < 2:
        raise ValueError("pass budget v must be >= 2")
    if _qr == "chol" and _checks is None:
        _qr = "householder"  # the CholeskyQR decline flag needs a caller that resolves it
    checks = _checks if _checks is not None else RankChecks()
    m, n = a.shape
    dev = a.device
    passes = 0
    basis = None
    if v % 2 == 0:
        om = core.omega(seed, m, l, dev)
        x = a.rmatmul(om)
        passes += 1
        if v == 2:
            basis = qr_basis_(x, checks, _qr)
            if _checks is None:
                checks.raise_if_collapsed()
            return RangeBasis(basis, passes)
        w = lu_basis_(x, checks)
    else:
        w = core.omega(seed, n, l, dev)
    half = (v - 1) // 2
    for i in range(1, half + 1):
        w = lu_basis_(a.matmul(w), checks)
        passes += 1
        if i == half:
            basis = qr_basis_(a.rmatmul(w), checks, _qr)
        else:
            w = lu_basis_(a.rmatmul(w), checks)
        passes += 1
    if _checks is None:
        checks.raise_if_collapsed()
    return RangeBasis(basis, passes)


def power_basis_v(a, l, p, seed):
    """rlra/rangefinder.py:137-141: odd pass budget 2p + 1."""
    if p < 1:
        raise ValueError("p must be >= 1: no products means no basis")
    return general_power_basis_v(a, l, 2 * p + 1, seed)


def final_sketch_lu_(y, checks):
    """rlra/rangefinder.py:129-132 (destroys y): SketchLU of the last sketch."""
    from .kernels import plu_

    f = plu_(y)
    checks.add(f.nonzero_diag, y.shape[1])
    return SketchLU(f.L, f.U, f.p)


def power_basis_q(a, l, p, seed):
    """rlra/rangefinder.py:86-103: column-space basis of (A A^T)^p A Omega with
    a Householder QR (K4) after every product; 2p + 1 passes."""
    a = as_accessor(a)
    _validate(a, l)
    if p < 0:
        raise ValueError("p must be >= 0")
    checks = RankChecks()
    om = core.omega(seed, a.shape[1], l, a.device)
    q = qr_basis_(a.matmul(om), checks)
    passes = 1
    for _ in range(p):
        q = qr_basis_(a.rmatmul(q), checks)
        q = qr_basis_(a.matmul(q), checks)
        passes += 2
    checks.raise_if_collapsed()
    return RangeBasis(q, passes)


def power_basis_lu_l(a, l, p, seed, *, _checks=None):
    """rlra/rangefinder.py:106-126: LU-stabilised sketch of A (A^T A)^p Omega
    for randlu -- (L, U, p) of the final pivoted LU (bit-exact GEPP, K3),
    interior renormalisations by the row-unpermuted L; 2p + 1 passes."""
    a = as_accessor(a)
    _validate(a, l)
    if p < 0:
        raise ValueError("p must be >= 0")
    checks = _checks if _checks is not None else RankChecks()
    om = core.omega(seed, a.shape[1], l, a.device)
    y = a.matmul(om)
    if p == 0:
        out = final_sketch_lu_(y, checks)
    else:
        w = lu_basis_(y, checks)
        for i in range(1, p + 1):
            w = lu_basis_(a.rmatmul(w), checks)
            y = a.matmul(w)
            if i == p:
                out = final_sketch_lu_(y, checks)
                break
            w = lu_basis_(y, checks)
    if _checks is None:
        checks.raise_if_collapsed()
    return out
