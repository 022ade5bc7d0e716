"""Fixed-rank PowerLU on device (rlra/fixedrank.py:18-155).

powerlu: v - 1 basis passes + the final G = A V_k pass, then the exact pivoted
assembly lu_from_projection (two bit-exact GEPPs, two DMMA GEMMs, one
transpose).  Output factors stay in HBM when the operand lives there, and come
back as NumPy arrays when the caller handed in host data (the reference's
return types).
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Any, NamedTuple

import numpy as np
import torch

from . import core, ops
from .device import DeviceMatrix, as_accessor, pass_engine, product_session
from .kernels import plu_, _copy, pinv_factor_
from .rangefinder import (RankChecks, final_sketch_lu_, general_power_basis_v, power_basis_lu_l,
                          power_basis_q)


@dataclass
class LowRankLU:
    """A[p, :][:, q] ~ L @ U (rlra/fixedrank.py:18-30).

    Fields are torch device tensors for device operands, NumPy arrays for host
    operands; ``to_numpy()`` converts."""

    p: Any
    q: Any
    L: Any
    U: Any
    rank: int

    def to_numpy(self):
        flds = [self.p, self.q, self.L, self.U]
        dev = [i for i, t in enumerate(flds) if isinstance(t, torch.Tensor)]
        for i, h in zip(dev, ops.to_numpy_many([flds[i] for i in dev])):
            flds[i] = h
        return LowRankLU(*flds, self.rank)

    @property
    def on_device(self):
        return isinstance(self.L, torch.Tensor)


class LowRankSVD(NamedTuple):
    """rlra/fixedrank.py:33-36: orthonormal U (m x r), S nonincreasing, V (n x r)."""

    U: Any
    S: Any
    V: Any

    def to_numpy(self):
        conv = lambda t: ops.to_numpy(t) if isinstance(t, torch.Tensor) and t.dim() == 2 else (
            t.cpu().numpy() if isinstance(t, torch.Tensor) else t)
        return LowRankSVD(conv(self.U), conv(self.S), conv(self.V))


def _validate_rank(a, k, q_os):
    """rlra/fixedrank.py:39-46."""
    m, n = a.shape
    if k < 1:
        raise ValueError("target rank must be >= 1")
    if q_os < 0:
        raise ValueError("oversampling must be >= 0")
    if k + q_os > min(m, n):
        raise ValueError(f"sketch width {k + q_os} exceeds min{(m, n)}")


def _host_input(a):
    return not (isinstance(a, torch.Tensor) or getattr(a, "is_device_accessor", False))


def lu_from_projection_(g, vk, checks=None):
    """rlra/fixedrank.py:136-146 on device; factors `g` IN PLACE.

    lu(G) -> (L1, U1, p); lu((U1 V^T)^T) -> (L2, U2, q); L = L1 U2^T, U = L2^T.
    """
    k = g.shape[1]
    prep_v = ops.tall_prep(vk, k)  # int8 residues of Vk, issued before the GEPP that hides their guard read
    f1 = plu_(g)  # L1 m x k, U1 k x k
    prep_l = ops.tall_prep(f1.L, k)
    bt = ops.tall_times(vk, f1.U, prep_v, ts=True)  # (U1 Vk^T)^T = Vk U1^T, n x k
    del prep_v
    f2 = plu_(bt)  # L2 n x k, U2 k x k
    big_l = ops.tall_times(f1.L, f2.U, prep_l, ts=True)  # L1 U2^T
    big_u = ops.transpose(f2.L)  # L2^T
    return LowRankLU(p=f1.p, q=f2.p, L=big_l, U=big_u, rank=k)


def lu_from_projection(g, vk):
    """Non-destructive, host-or-device wrapper of lu_from_projection_."""
    host = not isinstance(g, torch.Tensor)
    dev = ops.check_device()
    gd = ops.from_numpy(g, dev) if host else _copy(g)
    vd = ops.from_numpy(vk, dev) if not isinstance(vk, torch.Tensor) else vk
    f = lu_from_projection_(gd, vd)
    return f.to_numpy() if host else f


# Final basis of powerlu: "chol" (CholeskyQR2 + Householder fallback) or "householder".
POWERLU_QR = os.environ.get("RLRA_B200_POWERLU_QR", "chol")


def powerlu(a, k, q_os=10, v=3, seed=0):
    """Pass-parameterised randomized LU (rlra/fixedrank.py:120-133).  A
    distributed.ShardedMatrix runs the row-sharded multi-GPU algorithm."""
    if getattr(a, "is_sharded", False):
        from .distributed import api_powerlu

        return api_powerlu(a, k, q_os, v, seed)
    host = _host_input(a)
    a = as_accessor(a)
    _validate_rank(a, k, q_os)
    if v < 2:
        raise ValueError("pass budget v must be >= 2")
    checks = RankChecks()
    with product_session(a):
        basis = general_power_basis_v(a, k + q_os, v, seed, _checks=checks, _qr=POWERLU_QR)
        vk = basis.V[:, :k]
        g = a.matmul(vk)
        f = lu_from_projection_(g, vk)
        declined = checks.cholqr_declined()  # the only mid-call host sync, after all the work is queued
        if declined is not None and declined[0]:  # rare: redo the final basis by Householder, then G and LU
            from .rangefinder import qr_basis_

            v_h = qr_basis_(declined[1], checks, "householder")
            vk = v_h[:, :k]
            f = lu_from_projection_(a.matmul(vk), vk)
    checks.raise_if_collapsed()
    return f.to_numpy() if host else f


# The comparison baselines run their products on the native FP64 DMMA GEMM:
# their exact-zero rank checks (rlra/rangefinder.py:55-64, and the final
# sketch LU of randlu) see DGEMM-style rounding noise on exactly low-rank
# inputs, like the reference's BLAS, where the exact integer arithmetic of the
# int8 emulation can cancel a trailing pivot to exactly 0.0.
BASELINE_PASS = os.environ.get("RLRA_B200_BASELINE_PASS", "dmma")


def randsvd(a, k, q_os=10, p=1, seed=0, truncate=False):
    """Randomized SVD with QR-reorthogonalised power iteration
    (rlra/fixedrank.py:49-76): 2p + 2 passes.

    B = Q^T A (l x n) is formed as B^T = A^T Q (one pass) and reduced on device:
    B^T = Q2 R2 (Householder, K4), R2^T = Ub S Vr^T (one-sided Jacobi,
    csrc/svd.cu), so B = Ub S (Q2 Vr)^T and U = Q Ub, V = Q2 Vr -- the SVD
    np.linalg.svd(B) returns, up to the signs of singular-vector pairs."""
    host = _host_input(a)
    a = as_accessor(a)
    _validate_rank(a, k, q_os)
    with pass_engine(BASELINE_PASS), product_session(a):
        basis = power_basis_q(a, k + q_os, p, seed)
        bt = a.rmatmul(basis.V)  # n x l = (Q^T A)^T, one pass
    qr = ops.QR(bt)
    _, r2 = ops.lu_extract(qr.r_view(), want_l=False)  # R2: upper triangle of the packed QR
    r2t = ops.transpose(r2)
    ub, s, vr, _ = ops.svd_jacobi(r2t)
    u = ops.matmul(basis.V, ub)
    v = ops.matmul(qr.q(), vr)
    out = LowRankSVD(u[:, :k], s[:k], v[:, :k]) if truncate else LowRankSVD(u, s, v)
    if host:
        torch.cuda.synchronize()
        return out.to_numpy()
    return out


def _assemble_from_sketch_lu(a, sk, k):
    """rlra/fixedrank.py:108-117: pinv-based assembly of randlu."""
    ly = sk.L[:, :k]
    qr = pinv_factor_(ly)  # IllPosedPseudoinverse on a rank-deficient truncated sketch
    qy = qr.q()
    c = a.rmatmul(ops.apply_inv_row_perm(sk.p, qy))  # n x k, one pass
    x = ops.transpose(c)  # C^T, k x n
    ops.trsm_un_(qr.r_view(), x)  # B = R^{-1} C^T
    lb = plu_(ops.transpose(x))  # column pivoting through B^T
    big_l = ops.matmul(ly, lb.U, tb=True)
    return LowRankLU(p=sk.p, q=lb.p, L=big_l, U=ops.transpose(lb.L), rank=k)


def randlu(a, k, q_os=10, p=1, seed=0):
    """Randomized LU (rlra/fixedrank.py:79-91): LU-stabilised sketch,
    truncation to k, pivoted assembly; 2p + 2 passes."""
    host = _host_input(a)
    a = as_accessor(a)
    _validate_rank(a, k, q_os)
    checks = RankChecks()
    with pass_engine(BASELINE_PASS), product_session(a):
        sk = power_basis_lu_l(a, k + q_os, p, seed, _checks=checks)
        checks.raise_if_collapsed()
        f = _assemble_from_sketch_lu(a, sk, k)
    return f.to_numpy() if host else f


def randlu_noreorth(a, k, q_os=10, p=1, seed=0):
    """randlu on the raw chain A (A^T A)^p Omega (rlra/fixedrank.py:94-107)."""
    host = _host_input(a)
    a = as_accessor(a)
    _validate_rank(a, k, q_os)
    checks = RankChecks()
    with pass_engine(BASELINE_PASS), product_session(a):
        t = core.omega(seed, a.shape[1], k + q_os, a.device)
        for _ in range(p):
            t = a.rmatmul(a.matmul(t))
        sk = final_sketch_lu_(a.matmul(t), checks)
        checks.raise_if_collapsed()
        f = _assemble_from_sketch_lu(a, sk, k)
    return f.to_numpy() if host else f


def range_agreement(f1, f2):
    """Largest principal angle between the permuted L ranges
    (rlra/fixedrank.py:158-173; host validation metric, like reconstruct)."""
    f1 = f1.to_numpy() if isinstance(f1, LowRankLU) and f1.on_device else f1
    f2 = f2.to_numpy() if isinstance(f2, LowRankLU) and f2.on_device else f2
    if f1.L.shape[0] != f2.L.shape[0]:
        raise ValueError("row dimensions differ")
    if f1.rank != f2.rank:
        raise ValueError(f"rank mismatch: {f1.rank} vs {f2.rank}")

    def basis(f):
        x = np.empty_like(f.L)
        x[np.asarray(f.p), :] = f.L
        return np.linalg.qr(x)[0]

    q1, q2 = basis(f1), basis(f2)
    c = q1.T @ q2
    cos_min = np.linalg.svd(c, compute_uv=False)[-1]
    if cos_min ** 2 <= 0.5:
        return float(np.arccos(np.clip(cos_min, -1.0, 1.0)))
    sin_max = np.linalg.svd(q2 - q1 @ c, compute_uv=False)[0]
    return float(np.arcsin(np.clip(sin_max, -1.0, 1.0)))


def reconstruct(f):
    """rlra/fixedrank.py:149-155 (host; validation only)."""
    f = f.to_numpy() if isinstance(f, LowRankLU) else f
    r = f.L @ f.U
    out = np.empty_like(r)
    out[np.ix_(f.p, f.q)] = r
    return out
