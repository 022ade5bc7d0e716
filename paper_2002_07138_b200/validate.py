"""Validation metric at device scale:
||A[p, :][:, q] - L U||_F / ||A||_F (rlra/fixedrank.py:149-155 with
rlra/core.py:56-65) in column blocks on the GPU -- the reference's
`reconstruct` materialises m x n twice (137 GB at C5).  Per block, L U (m x w)
comes from the DMMA GEMM and the fused K9 kernel (csrc/misc.cu
resid_sumsq_kernel) gathers A's columns q through p, differences and sums the
squares in double-double, one partial per column; one fixed-order final sum.
Validation only: not on the factorization path."""

from __future__ import annotations

import math

import torch

from . import _native, ops


def rel_err_device(a, f, block=2048):
    """a: column-major device tensor (m x n); f: LowRankLU with device or host
    factors.  Returns the relative Frobenius reconstruction error (float)."""
    dev = a.device
    a = ops.as_fmat(a)
    t = lambda x: x if isinstance(x, torch.Tensor) else ops.from_numpy(x, dev) if getattr(x, "ndim", 1) == 2 \
        else torch.as_tensor(x, device=dev)
    L, U = t(f.L), t(f.U)
    p = torch.as_tensor(f.p, device=dev, dtype=torch.int64).contiguous()
    q = torch.as_tensor(f.q, device=dev, dtype=torch.int64).contiguous()
    m, n = a.shape
    if m == 0 or n == 0:
        return 0.0
    partial = torch.empty(2 * max(n, 1), dtype=torch.float64, device=dev)
    st = ops._stream(dev)
    for c0 in range(0, n, block):
        c1 = min(n, c0 + block)
        lu = ops.matmul(L, U[:, c0:c1])  # m x w
        ops._call("rlra_b200_resid_sumsq_block", dev, ops.ptr(a), ops.ld_of(a), m, ops.ptr(p),
                  ops.ptr(q) + 8 * c0, c1 - c0, ops.ptr(lu), ops.ld_of(lu), ops.ptr(partial) + 16 * c0, st)
    num = torch.empty(1, dtype=torch.float64, device=dev)
    ops._call("rlra_b200_dd_finish", dev, ops.ptr(partial), n, ops.ptr(num), st)
    den = ops.sumsq(a)
    return math.sqrt(float(num.item())) / math.sqrt(float(den.item()))
