"""Single-pass randomized LU over column-streamed matrices on device
(rlra/singlepass.py:99-144).

stream_sketch: one sweep, each panel read once; per panel G_j = panel^T Omega
(DMMA TN) written straight into its rows of G, then H += panel G_j (DMMA NN,
beta = 1) while the panel is still L2-resident, ascending column order like
the reference.  single_pass_lu: bit-exact GEPP of H, Householder QR of G with
the pinv rank test, blocked TRSM, one more GEMM, GEPP of T, and the assembly.
"""

from __future__ import annotations

from typing import NamedTuple

import torch

from . import core, ops
from .device import DEFAULT_PANEL, DenseColumnStream, DeviceColumnStream
from .fixedrank import LowRankLU
from .kernels import pinv_transpose_apply, plu_


class SketchPair(NamedTuple):
    G: torch.Tensor  # n x k
    H: torch.Tensor  # m x k


def stream_sketch(stream, k, seed, panel=DEFAULT_PANEL):
    """rlra/singlepass.py:99-120."""
    m, n = stream.shape
    if not 1 <= k <= min(m, n):
        raise ValueError(f"k={k} outside 1..min{(m, n)}")
    dev = getattr(stream, "device", None) or ops.check_device()
    om = core.omega(seed, m, k, dev)
    g = ops.fmat(n, k, dev)
    h = ops.fmat(m, k, dev, zero=True)
    count = 0
    for j0, block in stream.panels(panel):
        if not isinstance(block, torch.Tensor):
            block = ops.from_numpy(block, dev)
        w = block.shape[1]
        gb = g[j0:j0 + w, :]
        ops.gemm(block, om, gb, ta=True)  # G(j0:j0+w, :) = panel^T Omega
        ops.gemm(block, gb, h, beta=1.0)  # H += panel G_j
        count += w
    if count != n:
        raise ValueError(f"stream delivered {count} columns, expected {n}")
    return SketchPair(g, h)


def single_pass_lu(stream, k, seed, q_os=0, panel=DEFAULT_PANEL):
    """rlra/singlepass.py:123-144."""
    host = not isinstance(stream, DeviceColumnStream)  # host streams return NumPy factors
    l = k + q_os
    g, h = stream_sketch(stream, l, seed, panel=panel)
    f1 = plu_(h)  # L1 m x l, U1 l x l, p
    t = pinv_transpose_apply(g, ops.transpose(f1.U))  # (G^T)^+ U1^T
    f2 = plu_(t)  # L2 n x l, U2, q
    big_l = ops.matmul(f1.L, f2.U, tb=True)
    big_u = ops.transpose(f2.L)
    if q_os:
        big_l = big_l[:, :k]
        big_u = big_u[:k, :]
    f = LowRankLU(p=f1.p, q=f2.p, L=big_l, U=big_u, rank=k)
    return f.to_numpy() if host else f
