"""Validation metric at device scale (SURVEY.md §8(f) row 3, K9 scope):
||A[p, :][:, q] - L U||_F / ||A||_F (rlra/fixedrank.py:149-155 with
rlra/core.py:56-65) evaluated in column blocks on the GPU -- the reference's
`reconstruct` materialises m x n twice (137 GB at C5).  L U blocks come from
the DMMA GEMM; the permuted-A gather, difference and norms use torch as
plumbing.  Validation only: not on the factorization path."""

from __future__ import annotations

import math

import torch

from . import ops


def rel_err_device(a, f, block=2048):
    """a: column-major device tensor (m x n); f: LowRankLU with device or host
    factors.  Returns the relative Frobenius reconstruction error (float)."""
    dev = a.device
    t = lambda x: x if isinstance(x, torch.Tensor) else ops.from_numpy(x, dev) if getattr(x, "ndim", 1) == 2 \
        else torch.as_tensor(x, device=dev)
    L, U = t(f.L), t(f.U)
    p = torch.as_tensor(f.p, device=dev, dtype=torch.int64)
    q = torch.as_tensor(f.q, device=dev, dtype=torch.int64)
    m, n = a.shape
    num = torch.zeros((), dtype=torch.float64, device=dev)
    for c0 in range(0, n, block):
        c1 = min(n, c0 + block)
        lu = ops.matmul(L, U[:, c0:c1])  # m x w
        ablk = a[:, q[c0:c1]][p, :]  # gathered A[p, q[c0:c1]]
        d = ablk - lu
        num += (d * d).sum()
    den = ops.sumsq(a)
    return math.sqrt(float(num)) / math.sqrt(float(den.item()))
