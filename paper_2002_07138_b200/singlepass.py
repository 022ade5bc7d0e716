"""Single-pass randomized LU over column-streamed matrices on device
(rlra/singlepass.py:99-144).

stream_sketch: one sweep, each panel read once, ascending column order like
the reference; per panel G_j = panel^T Omega written straight into its rows of
G, then H += panel G_j.  Both products run on the int8 tensor cores (Ozaki-II,
csrc/ozaki.cu) from ONE residue set of the panel (TN, then NN with the CRT
adding into H); panels are consumed in sweep panels of up to SWEEP_PANEL
columns (a multiple of the caller's width) so the per-panel fixed costs stay
small -- G is unchanged by the grouping, H sees one rounding per sweep panel
instead of per panel.  DMMA when the int8 engine does not apply.  single_pass_lu: bit-exact GEPP of H, Householder QR of G with
the pinv rank test, blocked TRSM, one more GEMM, GEPP of T, and the assembly.
"""

from __future__ import annotations

from typing import NamedTuple

import torch

import os

from . import core, ops
from .device import DEFAULT_PANEL, PASS_GEMM, DenseColumnStream, DeviceColumnStream
from .fixedrank import LowRankLU
from .kernels import pinv_transpose_apply, plu_


class SketchPair(NamedTuple):
    G: torch.Tensor  # n x k
    H: torch.Tensor  # m x k


# Wider sweep panels amortise the per-panel CRT of H (m x l, read-modify-write)
# and the panel prologue: C4 (50000^2) 58.4 ms at 2 GB panels, 52.6 at 4 GB,
# 49.9 at 8 GB (profiles/r02b_c4_sweep_width.txt); 4 GB keeps a host stream's
# 3 pinned + 3 device slots at 12 GB each side.
SWEEP_PANEL = int(os.environ.get("RLRA_B200_SWEEP_PANEL", "16384"))
SWEEP_PANEL_BYTES = int(os.environ.get("RLRA_B200_SWEEP_BYTES", str(4 << 30)))  # one sweep panel of float64 (host streams keep 3 pinned + 3 device slots)
# The int8 engine's normwise error equals DGEMM's but it is not exact on
# sparse/identity panels (B is rounded relative to its column norm), which
# the reference's bitwise identity-stream property (pkg/tests/
# test_singlepass.py:15-24) relies on; small sweeps keep the native DMMA.
SWEEP_OZ_MIN_ELEMS = int(os.environ.get("RLRA_B200_SWEEP_OZ_MIN", str(1 << 24)))


def sweep_width(m, panel):
    """Columns per sweep panel: a multiple of the caller's width, <= SWEEP_PANEL
    columns and <= SWEEP_PANEL_BYTES (identical for every stream type, so host
    and device streams give bit-identical sketches)."""
    if panel < 1:
        raise ValueError("panel width must be >= 1")
    cap = min(SWEEP_PANEL, max(1, SWEEP_PANEL_BYTES // (8 * max(int(m), 1))))
    return panel * max(1, cap // panel)


def stream_sketch(stream, k, seed, panel=DEFAULT_PANEL):
    """rlra/singlepass.py:99-120 (a distributed.ShardedMatrix as the stream:
    the row-sharded sweep)."""
    if getattr(stream, "is_sharded", False):
        from .distributed import api_stream_sketch

        return api_stream_sketch(stream, k, seed, panel)
    m, n = stream.shape
    if not 1 <= k <= min(m, n):
        raise ValueError(f"k={k} outside 1..min{(m, n)}")
    dev = getattr(stream, "device", None) or ops.check_device()
    om = core.omega(seed, m, k, dev)
    g = ops.fmat(n, k, dev)
    h = ops.fmat(m, k, dev, zero=True)
    oz = PASS_GEMM == "oz" and 0 < m <= ops.OZ_BLOCK_K and k <= 4096 and m * n >= SWEEP_OZ_MIN_ELEMS
    count = 0
    om_ws, om_w = None, -1  # Omega's residues (the TN product's skinny operand) are the same for every panel
    for j0, block in stream.panels(sweep_width(m, panel) if oz else panel):
        if not isinstance(block, torch.Tensor):
            block = ops.from_numpy(block, dev)
        w = block.shape[1]
        gb = g[j0:j0 + w, :]
        if oz:
            with ops.label("sweep_oz"):
                prep = ops.OzPrep(block)  # residues of the panel, read once
                # G(j0:j0+w, :) = panel^T Omega; panels of equal width share one workspace layout
                _, ws_ = prep.gemm(om, trans=True, out=gb, keep_ws=True, b_ws=om_ws if w == om_w else None)
                if ws_ is not None:  # None: the guard sent this panel to the FP64 GEMM
                    om_ws, om_w = ws_, w
                prep.gemm(gb, out=h, add=True)  # H += panel G_j
        else:
            ops.gemm(block, om, gb, ta=True)  # G(j0:j0+w, :) = panel^T Omega
            ops.gemm(block, gb, h, beta=1.0)  # H += panel G_j
        count += w
    if count != n:
        raise ValueError(f"stream delivered {count} columns, expected {n}")
    return SketchPair(g, h)


def single_pass_lu(stream, k, seed, q_os=0, panel=DEFAULT_PANEL):
    """rlra/singlepass.py:123-144 (a distributed.ShardedMatrix as the stream:
    the row-sharded sweep, every rank gets the factors)."""
    if getattr(stream, "is_sharded", False):
        from .distributed import api_single_pass_lu

        return api_single_pass_lu(stream, k, seed, q_os, panel)
    host = not isinstance(stream, DeviceColumnStream)  # host streams return NumPy factors
    l = k + q_os
    g, h = stream_sketch(stream, l, seed, panel=panel)
    f1 = plu_(h)  # L1 m x l, U1 l x l, p
    prep_l = ops.tall_prep(f1.L, l)  # for L1 U2^T below; the pinv and the second GEPP hide its guard read
    t = pinv_transpose_apply(g, ops.transpose(f1.U))  # (G^T)^+ U1^T
    f2 = plu_(t)  # L2 n x l, U2, q
    big_l = ops.tall_times(f1.L, f2.U, prep_l, ts=True)
    big_u = ops.transpose(f2.L)
    if q_os:
        big_l = big_l[:, :k]
        big_u = big_u[:k, :]
    f = LowRankLU(p=f1.p, q=f2.p, L=big_l, U=big_u, rank=k)
    return f.to_numpy() if host else f
