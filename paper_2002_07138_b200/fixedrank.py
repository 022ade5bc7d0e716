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
from typing import Any

import numpy as np
import torch

from . import ops
from .device import DeviceMatrix, as_accessor, product_session
from .kernels import plu_, _copy
from .rangefinder import RankChecks, general_power_basis_v


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
        conv = lambda t: ops.to_numpy(t) if isinstance(t, torch.Tensor) else t
        torch.cuda.synchronize() if self.on_device else None
        return LowRankLU(conv(self.p), conv(self.q), conv(self.L), conv(self.U), self.rank)

    @property
    def on_device(self):
        return isinstance(self.L, torch.Tensor)


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
    f1 = plu_(g)  # L1 m x k, U1 k x k
    bt = ops.matmul(vk, f1.U, tb=True)  # (U1 Vk^T)^T = Vk U1^T, n x k
    f2 = plu_(bt)  # L2 n x k, U2 k x k
    big_l = ops.matmul(f1.L, f2.U, tb=True)  # L1 U2^T
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
    """Pass-parameterised randomized LU (rlra/fixedrank.py:120-133)."""
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
    checks.raise_if_collapsed()
    return f.to_numpy() if host else f


def reconstruct(f):
    """rlra/fixedrank.py:149-155 (host; validation only)."""
    f = f.to_numpy() if isinstance(f, LowRankLU) else f
    r = f.L @ f.U
    out = np.empty_like(r)
    out[np.ix_(f.p, f.q)] = r
    return out
