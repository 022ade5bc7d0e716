"""Fixed-precision PowerLU_FP with blocked adaptive rank (rlra/fixedprec.py).

The residual energy E = ||A||_F^2 - sum_j ||A v_j||^2 is tracked by
subtraction exactly like the reference; the energies themselves are computed
on device with compensated deterministic reductions (K2b for ||A||_F^2, K8 for
the column energies of G), and the l-long block/column scan runs on the host
with the reference's formulas (block energy = fro_norm(block)**2 =
sqrt(sum)**2, refinement by per-column `col @ col`).
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, replace
from typing import Any

import numpy as np
import torch

from . import ops
from .device import as_accessor, product_session
from .errors import NotConverged, Unsatisfiable
from .fixedrank import _host_input, lu_from_projection_
from .kernels import _copy
from .rangefinder import RankChecks, general_power_basis_v


@dataclass
class AdaptiveOutcome:
    """rlra/fixedprec.py:19-25."""

    rank: int
    V: Any  # n x rank, orthonormal
    G: Any  # m x rank, G = A @ V
    residual_energy: float
    converged: bool


@dataclass(frozen=True)
class PrecisionParams:
    """Tolerance eps, block size b, sketch width l (multiple of b), passes v
    (rlra/fixedprec.py:28-45, same validation)."""

    eps: float
    b: int
    l: int
    v: int

    def __post_init__(self):
        if not 0.0 < self.eps <= 1.0:
            raise ValueError(f"eps={self.eps} outside (0, 1]")
        if self.b < 1:
            raise ValueError("block size must be >= 1")
        if self.l < self.b or self.l % self.b:
            raise ValueError(f"sketch width {self.l} is not a positive multiple of {self.b}")
        if self.v < 2:
            raise ValueError("pass budget v must be >= 2")


def default_width(b, m, n):
    """rlra/fixedprec.py:48-54."""
    w = min(50 * b, min(m, n))
    w -= w % b
    if w < b:
        raise ValueError(f"block size {b} exceeds min{(m, n)}")
    return w


def refine_rank(g, e_in, acc, block_start, b):
    """rlra/fixedprec.py:97-110.  ``g`` is the matrix G (device tensor or
    ndarray); its column energies are computed on device for device tensors."""
    if isinstance(g, torch.Tensor):
        energy = ops.colsumsq(g[:, block_start:block_start + b]).cpu().numpy()
        energy = np.concatenate([np.zeros(block_start), energy])
    else:
        g = np.asarray(g, dtype=np.float64)
        energy = np.zeros(block_start + b)
        for j in range(b):
            col = g[:, block_start + j]
            energy[block_start + j] = float(col @ col)
    return _refine_from_energies(energy, e_in, acc, block_start, b)


def _refine_from_energies(col_energy, e_in, acc, block_start, b):
    """The per-column loop of rlra/fixedprec.py:97-110 over column energies."""
    e = e_in
    for j in range(b):
        e -= float(col_energy[block_start + j])
        if e <= acc:
            return block_start + j + 1, e
    return block_start + b, e


def scan_energies(total, col_energy, eps, b, l):
    """The block scan of rlra/fixedprec.py:73-94 given ||A||_F^2 and the
    per-column energies of G; returns (rank, residual, converged)."""
    acc = eps**2 * total
    e = total
    for t1 in range(0, l, b):
        e_before = e
        e -= math.sqrt(float(np.sum(col_energy[t1:t1 + b]))) ** 2
        if e <= acc:
            rank, e_out = _refine_from_energies(col_energy, e_before, acc, t1, b)
            return rank, max(e_out, 0.0), True
    return l, max(e, 0.0), False


# Final basis of powerlu_fp: "chol" (CholeskyQR2 / shifted CholeskyQR3, the
# Householder redo when it declines) or "householder".
POWERLU_FP_QR = os.environ.get("RLRA_B200_POWERLU_FP_QR", "chol")


def _g_and_energies(a, v):
    """G = A V and its column energies (rlra/fixedprec.py:71-80): fused with
    the product where the accessor offers it (DeviceMatrix: the CRT step of the
    int8 pass), else the K8 reduction over G."""
    fused = getattr(a, "matmul_with_energies", None)
    if fused is not None:
        return fused(v)
    g = a.matmul(v)
    return g, ops.colsumsq(g)


def _adaptive(a, params, seed):
    m, n = a.shape
    if params.l > min(m, n):
        raise ValueError(f"sketch width {params.l} exceeds min{(m, n)}")
    checks = RankChecks()
    with product_session(a):
        basis = general_power_basis_v(a, params.l, params.v, seed, _checks=checks, _qr=POWERLU_FP_QR)
        V = basis.V
        g, energies = _g_and_energies(a, V)
        declined = checks.cholqr_declined()  # one host round trip (the counts ride along)
        if declined is not None and declined[0]:  # rare: Householder basis, then G again
            from .rangefinder import qr_basis_

            V = qr_basis_(declined[1], checks, "householder")
            g, energies = _g_and_energies(a, V)
        fro2 = a.fro_norm_sq_device()  # inside the session: fused into the pass's norms read
    checks.raise_if_collapsed()
    host = torch.cat([fro2, energies]).cpu().numpy()
    # total = fro_norm(a) ** 2 (rlra/fixedprec.py:72): norm then square, as there
    total = math.sqrt(float(host[0])) ** 2
    rank, resid, conv = scan_energies(total, host[1:], params.eps, params.b, params.l)
    return AdaptiveOutcome(rank, V[:, :rank], g[:, :rank], resid, conv)


def adaptive_rank(a, params, seed):
    """rlra/fixedprec.py:57-94."""
    if getattr(a, "is_sharded", False):
        from .distributed import api_adaptive_rank

        return api_adaptive_rank(a, params, seed)
    host = _host_input(a)
    out = _adaptive(as_accessor(a), params, seed)
    if host:
        out = AdaptiveOutcome(out.rank, ops.to_numpy(out.V), ops.to_numpy(out.G),
                              out.residual_energy, out.converged)
    return out


def powerlu_fp(a, params, seed):
    """rlra/fixedprec.py:152-163: (LowRankLU, AdaptiveOutcome) or NotConverged."""
    if getattr(a, "is_sharded", False):
        from .distributed import api_powerlu_fp

        return api_powerlu_fp(a, params, seed)
    host = _host_input(a)
    out = _adaptive(as_accessor(a), params, seed)
    if not out.converged:
        if host:
            out = AdaptiveOutcome(out.rank, ops.to_numpy(out.V), ops.to_numpy(out.G),
                                  out.residual_energy, out.converged)
        raise NotConverged(out)
    f = lu_from_projection_(_copy(out.G), out.V)
    if host:
        f = f.to_numpy()
        out = AdaptiveOutcome(out.rank, ops.to_numpy(out.V), ops.to_numpy(out.G),
                              out.residual_energy, out.converged)
    return f, out


def restart_policy(prev, params, max_width):
    """rlra/fixedprec.py:166-181 (host policy, unchanged)."""
    if prev.converged:
        raise ValueError("restart on a converged outcome makes no sense")
    cap = max_width - max_width % params.b
    if cap < params.b or params.l >= cap:
        raise Unsatisfiable(f"sketch width {params.l} already at cap {cap} without converging")
    return replace(params, l=min(2 * params.l, cap))
