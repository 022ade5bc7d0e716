"""Multi-GPU PowerLU: A row-sharded across the ranks of one node, one process
per GPU, torch.distributed over NCCL (NVLink 5 / NVSwitch) for the exchanges
(SURVEY.md §8(e)).

Per pass (rlra/rangefinder.py:144-176 control flow, unchanged):
  Y = A W     local rows only (W replicated)            no communication
  Z = A^T Y   local partial A_i^T Y_i, then all-reduce   n x l doubles
  ||A||_F^2   local compensated sum, then all-reduce     1 double
  column energies of G: local, then all-reduce           l doubles
Sketch factorizations:
  interior LU of the row-sharded Y: TSLU (tournament pivoting, SURVEY.md
  §8(e)) -- local GEPP of Y_i names l candidate rows per rank, one all-gather
  of the world*l x l candidates, a redundant GEPP of those gives U, and
  W_i = Y_i U^{-1} locally.  Any pivoting gives W = Y U^{-1} with U upper
  triangular, so range(W) is that of the exact GEPP's P^T L and the final QR
  absorbs the difference (V equal up to column signs and rounding); traffic is
  world*l*l doubles instead of the whole m x l sketch.  RLRA_B200_DIST_INTERIOR
  =gather selects the all-gathered exact GEPP instead.
  final LU of G: EXACT GEPP on the all-gathered matrix (every rank
  redundantly, bit-exact kernel), so p and q are those of the single-GPU /
  reference algorithm; LU / QR of the replicated n x l sketches run
  redundantly with no communication.

Single-pass LU (rlra/singlepass.py:99-144) over the same row shards: per sweep
panel J, G_J = sum_i A_i(:, J)^T Omega_i is a local partial product followed
by an all-reduce (w x l), issued asynchronously so it overlaps the next
panel's partial product; H_i += A_i(:, J) G_J stays local (H row-sharded).
H is all-gathered for its exact GEPP; G is replicated for the QR / TRSM / LU.

The orchestration is written against a small ops interface so the same code
runs on CUDA tensors with NCCL (CudaOps, the product) and -- in the CPU test
suite only -- on CPU tensors with gloo and an oracle-backed ops object
(tests/test_distributed_gloo.py).
"""

from __future__ import annotations

import contextlib
import os
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from .errors import NotConverged, RankCollapse


def row_range(m, world, rank):
    """Contiguous, nearly equal row shards (the last ones may be shorter)."""
    per = -(-m // world)
    r0 = min(m, rank * per)
    return r0, min(m, r0 + per)


class CudaOps:
    """Product ops: librlra_b200 kernels on CUDA tensors."""

    def __init__(self, device):
        from . import ops as _ops

        self.o = _ops
        self.device = device

    def upload(self, a):
        return self.o.from_numpy(a, self.device)

    def empty(self, m, n):
        return self.o.fmat(m, n, self.device)

    def matmul(self, a, b, ta=False, tb=False):
        return self.o.matmul(a, b, ta=ta, tb=tb)

    def pass_prep(self, a):
        """Int8 residues of the local shard for the emulated pass products."""
        from .device import OZ_MAX_RESIDUE_BYTES, PASS_GEMM

        if PASS_GEMM != "oz" or min(a.shape) == 0:
            return None
        return self.o.oz_engine(a, OZ_MAX_RESIDUE_BYTES)

    def pass_matmul(self, a, prep, x, ta=False):
        if prep is not None and 0 < x.shape[1] <= 4096:
            return prep.gemm(x, trans=ta)
        return self.o.matmul(a, x, ta=ta)

    def zeros(self, m, n):
        return self.o.fmat(m, n, self.device, zero=True)

    # ---- row-sharded exact GEPP primitives (dist_getrf_; csrc/getrf.cu)
    def gepp_state(self, m, n):
        """piv (iota), zflag, ipiv, nonzero count and the getrf workspace."""
        o = self.o
        wsb = o._native.query("rlra_b200_getrf_workspace", m, n)
        return {"piv": o.iota(m, self.device),
                "zflag": torch.zeros(max(n, 1), dtype=torch.int32, device=self.device),
                "ipiv": torch.zeros(max(n, 1), dtype=torch.int64, device=self.device),
                "cnt": torch.zeros(1, dtype=torch.int64, device=self.device),
                "ws": torch.empty(max(wsb, 8), dtype=torch.uint8, device=self.device), "wsb": wsb}

    def getrf_block(self, panel, j0, nbo, stt):
        """Factor the gathered m x nbo panel (global columns [j0, j0+nbo)) in place."""
        o, m = self.o, panel.shape[0]
        base = o.ptr(panel) - 8 * j0 * o.ld_of(panel)  # virtual base: column j0 is the panel's first
        o._call("rlra_b200_getrf_block", self.device, base, o.ld_of(panel), m, j0, nbo, o.ptr(stt["piv"]),
                o.ptr(stt["zflag"]), o.ptr(stt["ipiv"]), o.ptr(stt["cnt"]), o.ptr(stt["ws"]), stt["wsb"],
                o._stream(self.device))

    def unit_lower_rows(self, local, pos0):
        """Rows [pos0, pos0 + rows) of a packed L\\U -> the same rows of the unit
        lower L (min(m, n) columns): entries left of the diagonal, 1 on it."""
        rows, n = local.shape
        out = self.o.fmat(rows, n, self.device)
        out.copy_(torch.tril(local, diagonal=pos0 - 1))
        lo, hi = max(0, pos0), min(pos0 + rows, n)
        if hi > lo:  # rows past the last column (most ranks' shards) have no diagonal entry
            d = torch.arange(lo, hi, device=self.device)
            out[d - pos0, d] = 1.0
        return out

    def ipiv_host(self, stt, j0, nbo):
        return stt["ipiv"][j0:j0 + nbo].cpu().tolist()

    def lu_trsm_rows(self, blk, j0, nbo, c0, c1, stt):
        """U12 = L11^-1 A12 in the block's gathered rows (nbo x n, global rows j0..)."""
        o = self.o
        o._call("rlra_b200_lu_trsm_rows", self.device, o.ptr(blk) - 8 * j0, o.ld_of(blk), j0, nbo, c0, c1,
                o.ptr(stt["zflag"]), o._stream(self.device))

    def lu_update_split(self, local, blk, j0, nbo, r_lo, c0, c1, stt):
        """local[r_lo:, c0:c1] -= local[r_lo:, j0:j0+nbo] U12 (U12 in blk)."""
        o = self.o
        o._call("rlra_b200_lu_update_split", self.device, o.ptr(local), o.ld_of(local), o.ptr(blk) - 8 * j0,
                o.ld_of(blk), j0, nbo, r_lo, local.shape[0], c0, c1, o.ptr(stt["zflag"]), o._stream(self.device))

    def sweep_width(self, m, panel):
        from .singlepass import sweep_width

        return sweep_width(m, panel) if self.sweep_oz(m, 1 << 30, 1) else panel

    def sweep_oz(self, m, n, k):
        from .device import PASS_GEMM
        from .singlepass import SWEEP_OZ_MIN_ELEMS

        return PASS_GEMM == "oz" and 0 < m <= self.o.OZ_BLOCK_K and k <= 4096 and m * n >= SWEEP_OZ_MIN_ELEMS

    def sweep_prep(self, block, oz):
        """Residues of one sweep panel (read once, both products), or None."""
        return self.o.OzPrep(block) if oz and min(block.shape) > 0 else None

    def sweep_products(self, block, prep, x, out, ta, add):
        """out = block^T x (ta) or out += block x (add) on the sweep engine."""
        if prep is not None:
            return prep.gemm(x, trans=ta, out=out, add=add)
        return self.o.gemm(block, x, out, ta=ta, beta=1.0 if add else 0.0)

    def pinv_transpose_apply(self, g, m_):
        from .kernels import pinv_transpose_apply

        return pinv_transpose_apply(g, m_)

    def getrf_(self, a):
        return self.o.getrf_(a)

    def lu_basis(self, lu, piv):
        return self.o.lu_basis(lu, piv)

    def lu_extract(self, lu):
        return self.o.lu_extract(lu)

    def qr_q(self, x):
        qr = self.o.QR(x)
        return qr.q(), self.o.count_nonzero_diag(qr.r_view())

    def qr_q_fast(self, x):
        """powerlu's final basis as on one GPU: CholeskyQR2, Householder when
        the Cholesky declines (rangefinder.qr_basis_ with method="chol")."""
        if x.shape[0] >= x.shape[1] and 0 < x.shape[1] <= self.o.cholqr_max_l():
            q, flag = self.o.cholqr2(x)
            if not int(flag.item()):
                return q, None
        return self.qr_q(x)

    def transpose(self, a):
        return self.o.transpose(a)

    def chol_inv(self, g, cond_limit, flag=None):
        """R^{-1} of chol(g) (upper, any l: blocked beyond the one-CTA kernel)
        and the device decline flag (csrc/cholqr.cu)."""
        l = g.shape[0]
        if flag is None:
            flag = torch.zeros(1, dtype=torch.int32, device=self.device)
        rinv = self.o.fmat(l, l, self.device)
        self.o.chol_inv_blocked(g, rinv, flag, cond_limit)
        return rinv, flag

    def shift_gram(self, g, n, flag):
        """sCholQR3's first step: flag an exactly zero column, g += s I."""
        l = g.shape[0]
        st = self.o._stream(self.device)
        self.o._call("rlra_b200_diag_ratio_flag", self.device, self.o.ptr(g), self.o.ld_of(g), l,
                     self.o.NO_COND_LIMIT, self.o.ptr(flag), st)
        self.o._call("rlra_b200_chol_shift_diag", self.device, self.o.ptr(g), self.o.ld_of(g), l,
                     self.o.SCHOL_C * (n * l + l * (l + 1)), st)

    def gram_identity_flag(self, g, flag):
        self.o.gram_identity_flag(g, flag)

    def cholqr_wide(self, l):
        return l > self.o.cholqr_max_l()

    def cholqr_ok(self, x):
        return x.shape[0] >= x.shape[1] > 0

    def qr_qr(self, x):
        """Householder Q (m x l) and R (l x l) of x (destroyed)."""
        qr = self.o.QR(x)
        _, r = self.o.lu_extract(qr.r_view(), want_l=False)
        return qr.q(), r

    def flag_value(self, flag):
        return int(flag.item())

    def nonzero_diag(self, r):
        return self.o.count_nonzero_diag(r)

    def sumsq(self, a):
        return self.o.sumsq(a)

    def colsumsq(self, a):
        return self.o.colsumsq(a)

    def gather_rows(self, x, idx):
        return self.o.as_fmat(x.index_select(0, idx))

    def right_solve_upper(self, x, u):
        """X U^{-1} (U upper l x l): U^{-1} by the K6 solve U X = I (l^3, small),
        then one DMMA GEMM over the tall X (the transposed TRSM took 3.4 ms on
        a 32768 x 544 shard, profiles/r02_scale_model_C5.json)."""
        if x.shape[0] == 0:
            return x
        l = u.shape[0]
        inv = self.o.fmat(l, l, self.device)
        inv.copy_(torch.eye(l, dtype=torch.float64, device=self.device))
        self.o.trsm_un_(u, inv)
        return self.o.matmul(x, inv)


@dataclass
class DistLU:
    """Factors of a distributed call: p, q, U replicated on every rank; L
    row-sharded by position -- this rank holds rows [l0, l1) of the m x k L
    (L = L1 U2^T is the largest GEMM of the assembly, 2 m k^2 flops: each rank
    forms only its block).  full_L() all-gathers it."""
    p: object
    q: object
    L: object
    U: object
    rank: int
    l0: int = 0
    l1: int = -1
    m: int = 0
    group: object = None
    ops: object = None

    @property
    def sharded(self):
        return self.l1 >= 0 and (self.l0, self.l1) != (0, self.m)

    def full_L(self):
        if not self.sharded:
            return self.L
        world = dist.get_world_size(self.group)
        k = self.L.shape[1]
        per = -(-self.m // world)
        buf = torch.zeros((k, per), dtype=self.L.dtype, device=self.L.device)
        if self.l1 > self.l0:
            buf[:, : self.l1 - self.l0].copy_(self.L.t())
        out = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(out, buf, group=self.group)
        full = self.ops.empty(self.m, k)
        for r in range(world):
            a0, a1 = row_range(self.m, world, r)
            if a1 > a0:
                full[a0:a1, :].copy_(out[r][:, : a1 - a0].t())
        return full


class ShardedMatrix:
    """Row shard A_i (rows [r0, r1) of the m x n operand) on this rank.

    Passing it to the drop-in API (powerlu, powerlu_fp, adaptive_rank,
    general_power_basis_v, single_pass_lu, stream_sketch -- the reference
    signatures, rlra/fixedrank.py:120, rlra/fixedprec.py:152, ...) runs the
    row-sharded algorithm over `group`; every rank gets the same factors.
    omega_fn(seed, rows, l) draws Omega (default: the device replay of
    rlra.core.gaussian)."""

    is_sharded = True

    def __init__(self, local, m, r0, r1, ops, group=None, omega_fn=None):
        self.local = local
        self.omega_fn = omega_fn
        self.m, self.n = int(m), int(local.shape[1])
        self.r0, self.r1 = r0, r1
        self.ops = ops
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.product_count = 0
        self._sessions = 0
        self._prep = None
        self._prep_built = False

    @contextlib.contextmanager
    def products(self):
        """Pass products of one driver call share the residues of A_i."""
        self._sessions += 1
        try:
            yield self
        finally:
            self._sessions -= 1
            if self._sessions == 0:
                self._prep, self._prep_built = None, False

    def _pass(self, x, ta):
        if not hasattr(self.ops, "pass_matmul"):
            return self.ops.matmul(self.local, x, ta=ta)
        prep = self._prep
        if not self._prep_built:
            prep = self.ops.pass_prep(self.local)
            if self._sessions > 0:
                self._prep, self._prep_built = prep, True
        return self.ops.pass_matmul(self.local, prep, x, ta=ta)

    @property
    def shape(self):
        return (self.m, self.n)

    # ---- passes
    def matmul(self, w):
        """Y_i = A_i W (W replicated n x w) -> local rows of Y."""
        self.product_count += 1
        return self._pass(w, False)

    def rmatmul(self, y_local):
        """Z = sum_i A_i^T Y_i -> replicated n x w (NCCL all-reduce)."""
        self.product_count += 1
        z = self._pass(y_local, True)
        # column-major (n, w) == contiguous (w, n) storage: reduce that view in place
        dist.all_reduce(z.t(), op=dist.ReduceOp.SUM, group=self.group)
        return z

    def fro_norm_sq(self):
        s = self.ops.sumsq(self.local).clone()
        dist.all_reduce(s, op=dist.ReduceOp.SUM, group=self.group)
        return s

    # ---- exchanges
    def gather_rows(self, y_local):
        """All-gather the row-sharded m x w matrix to every rank (column-major)."""
        w = y_local.shape[1]
        per = -(-self.m // self.world)
        # pad each shard to `per` rows; gather as (world, w, per) row-major blocks
        buf = torch.zeros((w, per), dtype=y_local.dtype, device=y_local.device)
        rows = self.r1 - self.r0
        if rows:
            buf[:, :rows].copy_(y_local.t())
        out = [torch.empty_like(buf) for _ in range(self.world)]
        dist.all_gather(out, buf, group=self.group)
        full = self.ops.empty(self.m, w)
        for r in range(self.world):
            a0, a1 = row_range(self.m, self.world, r)
            if a1 > a0:
                full[a0:a1, :].copy_(out[r][:, : a1 - a0].t())
        return full

    def local_rows(self, full):
        return full[self.r0:self.r1, :]


INTERIOR = os.environ.get("RLRA_B200_DIST_INTERIOR", "tslu")  # "tslu" | "gather" | "tslu_always" (also 1 rank)


def tslu_basis_rows(A, y_local, l):
    """Interior renormalisation of the row-sharded sketch by tournament
    pivoting; returns this rank's rows of W = Y U^{-1}."""
    ops = A.ops
    rows = y_local.shape[0]
    c = min(rows, l)
    dev = y_local.device
    cand = torch.zeros((l, l), dtype=torch.float64, device=dev)  # row-major candidate rows
    gidx = torch.full((l,), -1, dtype=torch.int64, device=dev)
    if rows:
        work = ops.empty(rows, l)
        work.copy_(y_local)
        piv, _ = ops.getrf_(work)
        sel = piv[:c].to(dev)
        cand[:c].copy_(y_local.index_select(0, sel))
        gidx[:c] = sel + A.r0
    cands = [torch.empty_like(cand) for _ in range(A.world)]
    idxs = [torch.empty_like(gidx) for _ in range(A.world)]
    dist.all_gather(cands, cand, group=A.group)
    dist.all_gather(idxs, gidx, group=A.group)
    full = ops.empty(A.world * l, l)
    full.copy_(torch.cat(cands, 0))
    _, cnt = ops.getrf_(full)  # redundant on every rank: identical U everywhere
    _check(cnt, l)
    _, u = ops.lu_extract(full)
    return ops.right_solve_upper(y_local, u)


def _check(count, requested):
    achieved = int(count.item())
    if achieved < requested:
        raise RankCollapse(achieved, requested)


LU_BLOCK = 32  # csrc/getrf.cu LU_NB


def _net_perm(j0, seq):
    """Net row permutation of the interchange sequence (row j0+q <-> seq[q],
    q ascending) as (touched positions, source positions)."""
    rows, src = [], {}
    for q, pr in enumerate(seq):
        jq = j0 + q
        if pr == jq:
            continue
        for r in (jq, pr):
            if r not in src:
                src[r] = r
                rows.append(r)
        src[jq], src[pr] = src[pr], src[jq]
    return rows, [src[r] for r in rows]


def _owned_rows(A, buf, positions):
    """Every rank gets the rows of `buf` (len(positions) x n) that their owners
    filled: all-gather, then each row from its owner's copy -- a summing
    all-reduce would turn -0.0 into +0.0 (bit-exactness includes zero signs)."""
    if A.world == 1:
        return buf
    send = buf.t().contiguous()  # column-major (rows, n) == row-major (n, rows)
    outs = [torch.empty_like(send) for _ in range(A.world)]
    dist.all_gather(outs, send, group=A.group)
    res = A.ops.empty(buf.shape[0], buf.shape[1])
    for t, pos in enumerate(positions):
        owner = _owner(A.m, A.world, pos)
        res[t].copy_(outs[owner].t()[t])
    return res


def _owner(m, world, pos):
    per = -(-m // world)
    return min(world - 1, pos // per) if per else 0


def dist_getrf_(A, local):
    """Exact GEPP (rlra/_lu_cython.pyx:14-55, bit-identical to the one-GPU
    kernel) of the row-sharded m x n matrix whose rows [A.r0, A.r1) this rank
    holds as `local` (factored in place: its rows of the packed L\\U, in the
    final row order).  Per 32-column block J:
      1. all-gather the panel's m x 32 columns (positions order);
      2. every rank factors it redundantly (getrf_block: same pivots everywhere);
      3. the block's interchanges move <= 64 full rows between ranks (one
         all-reduce of those rows);
      4. the block's 32 rows are all-reduced, U12 = L11^-1 A12 on every rank;
      5. each rank updates only its own rows (bit-exact update kernel).
    Communication per block: m*32 + 96*n doubles; no m x n gather, no
    replicated m x n factorization.  Returns (piv replicated int64[m], the
    n x n block rows of U replicated (rows 0..n of the packed factor), the
    nonzero-diagonal count)."""
    ops = A.ops
    m, n = A.m, local.shape[1]
    r0, r1 = A.r0, A.r1
    stt = ops.gepp_state(m, n)
    urows = ops.zeros(min(m, n), n)
    for j0 in range(0, min(m, n), LU_BLOCK):
        nbo = min(LU_BLOCK, min(m, n) - j0)
        panel = A.gather_rows(local[:, j0:j0 + nbo])
        ops.getrf_block(panel, j0, nbo, stt)
        rows, srcs = _net_perm(j0, ops.ipiv_host(stt, j0, nbo))
        if rows:  # full-row interchanges on the columns outside the block
            moved = ops.zeros(len(rows), n)
            for t, sp in enumerate(srcs):
                if r0 <= sp < r1:
                    moved[t].copy_(local[sp - r0])
            moved = _owned_rows(A, moved, srcs)
            for t, rp in enumerate(rows):
                if r0 <= rp < r1:
                    if j0 > 0:
                        local[rp - r0, :j0].copy_(moved[t, :j0])
                    if j0 + nbo < n:
                        local[rp - r0, j0 + nbo:].copy_(moved[t, j0 + nbo:])
        if r1 > r0:
            local[:, j0:j0 + nbo].copy_(panel[r0:r1])
        blk = ops.zeros(nbo, n)  # the block's rows j0..j0+nbo, all columns
        b0, b1 = max(r0, j0), min(r1, j0 + nbo)
        if b1 > b0:
            blk[b0 - j0:b1 - j0].copy_(local[b0 - r0:b1 - r0])
        blk = _owned_rows(A, blk, range(j0, j0 + nbo))
        if j0 + nbo < n:
            ops.lu_trsm_rows(blk, j0, nbo, j0 + nbo, n, stt)
            if b1 > b0:
                local[b0 - r0:b1 - r0, j0 + nbo:].copy_(blk[b0 - j0:b1 - j0, j0 + nbo:])
            lo = max(r0, j0 + nbo) - r0
            if lo < r1 - r0:
                ops.lu_update_split(local, blk, j0, nbo, lo, j0 + nbo, n, stt)
        urows[j0:j0 + nbo].copy_(blk)
    return stt["piv"], urows, stt["cnt"]


def _use_tslu(A, l):
    """Interior LU of a row-sharded sketch: TSLU at 4+ ranks or tall sketches
    (the all-gather of m x l and the replicated m x l GEPP grow with m, the
    tournament does not); the all-gathered exact GEPP at 2 ranks."""
    if INTERIOR == "tslu_always":
        return True
    if INTERIOR != "tslu" or A.world < 2:
        return False
    return A.world >= 4 or A.m > 131072


def general_power_basis_v(A: ShardedMatrix, l, v, seed, omega_fn, fast_qr=False):
    """rlra/rangefinder.py:144-176 over a row-sharded A.  omega_fn(seed, rows, l)
    returns the full Omega (bit-exact rlra.core.gaussian): a host array, or a
    device tensor (core.omega) that is sliced in place.  fast_qr: powerlu's
    final basis by CholeskyQR2 (as on one GPU)."""
    m, n = A.shape
    if not 1 <= l <= min(m, n):
        raise ValueError(f"sketch width l={l} outside 1..min{(m, n)}")
    if v < 2:
        raise ValueError("pass budget v must be >= 2")
    ops = A.ops

    def lu_basis_rows(y_local):
        if _use_tslu(A, l):
            return tslu_basis_rows(A, y_local, l)
        full = A.gather_rows(y_local)
        piv, cnt = ops.getrf_(full)
        _check(cnt, l)
        return A.local_rows(ops.lu_basis(full, piv))

    n_rows = A.shape[1]
    shard = SHARD_REPLICATED and _block_ok(A, n_rows, l)

    def lu_basis_repl(z):
        # the tournament only pays for very tall sketches: its local and
        # candidate GEPPs are latency bound like the replicated one
        # (profiles/r02_time_getrf.txt: 4096 x 544 and 32768 x 544 both ~2-4 ms)
        if shard and _use_tslu(A, l) and n_rows > REPL_TSLU_MIN_ROWS:
            return sharded_lu_basis(A, z, l)
        piv, cnt = ops.getrf_(z)
        _check(cnt, l)
        return ops.lu_basis(z, piv)

    def qr_basis(z):
        if shard and fast_qr:
            q, cnt = sharded_qr_basis(A, z)
        else:
            q, cnt = (ops.qr_q_fast if fast_qr and hasattr(ops, "qr_q_fast") else ops.qr_q)(z)
        if cnt is not None:
            _check(cnt, l)
        return q

    def omega_rows(rows, r0, r1):
        om = omega_fn(seed, rows, l)
        if isinstance(om, torch.Tensor):  # device Omega (core.omega): slice, no copy
            return om[r0:r1]
        return ops.upload(np.asfortranarray(om[r0:r1]))

    if v % 2 == 0:
        x = A.rmatmul(omega_rows(m, A.r0, A.r1))
        if v == 2:
            return qr_basis(x), 1
        w = lu_basis_repl(x)
    else:
        w = omega_rows(n, 0, n)
    half = (v - 1) // 2
    passes = 1 if v % 2 == 0 else 0
    basis = None
    for i in range(1, half + 1):
        w_rows = lu_basis_rows(A.matmul(w))
        passes += 1
        z = A.rmatmul(w_rows)
        passes += 1
        if i == half:
            basis = qr_basis(z)
        else:
            w = lu_basis_repl(z)
    return basis, passes


SHARD_L = os.environ.get("RLRA_B200_DIST_SHARD_L", "1") == "1"


def _assemble(A, l1, u2, l2, piv1, piv2, k, cut=None):
    """L = L1 U2^T (row block of this rank when SHARD_L), U = L2^T."""
    ops = A.ops
    m = l1.shape[0]
    if SHARD_L and A.world > 1:
        p0, p1 = row_range(m, A.world, A.rank)
        big_l = ops.matmul(l1[p0:p1], u2, tb=True)
    else:
        p0, p1 = 0, m
        big_l = ops.matmul(l1, u2, tb=True)
    big_u = ops.transpose(l2)
    if cut is not None:
        big_l, big_u = big_l[:, :cut], big_u[:cut, :]
    return DistLU(piv1, piv2, big_l, big_u, k, p0, p1, m, A.group, ops)


DIST_GEPP = os.environ.get("RLRA_B200_DIST_GEPP", "1") == "1"  # 0: all-gather + replicated exact GEPP


def _dist_lu(S, local):
    """Row-sharded exact GEPP of S (a ShardedMatrix over `local`, factored in a
    copy): (piv replicated, U (r x r upper, replicated), this rank's rows of the
    unit-lower L in final row order, nonzero-diagonal count)."""
    ops = S.ops
    work = ops.empty(local.shape[0], local.shape[1])
    work.copy_(local)
    piv, urows, cnt = dist_getrf_(S, work)
    _, u = ops.lu_extract(urows)
    return piv, u, ops.unit_lower_rows(work, S.r0), cnt


def _lu_factors_sharded(A, left_local, right_rows, k):
    """The two exact GEPPs of rlra/fixedrank.py:144-146 / singlepass.py:
    :134-136 without gathering the tall operand: LU(left) over A's row shards,
    the right operand (n x k) computed / sliced by row blocks, its LU sharded
    too; L = L1 U2^T by this rank's rows, U = L2^T (L2 all-gathered)."""
    piv1, u1, l1_rows, cnt = _dist_lu(A, left_local)
    n = right_rows.n_total
    c0, c1 = row_range(n, A.world, A.rank)
    bt_local = right_rows.rows(u1, c0, c1)
    B = ShardedMatrix(bt_local, n, c0, c1, A.ops, A.group)
    piv2, u2, l2_rows, _ = _dist_lu(B, bt_local)
    big_l = A.ops.matmul(l1_rows, u2, tb=True)
    l2 = B.gather_rows(l2_rows)
    big_u = A.ops.transpose(l2)
    return piv1, piv2, big_l, big_u, cnt


class _BtRows:
    """B^T = V_k U1^T (rlra/fixedrank.py:145) by row blocks."""

    def __init__(self, vk, ops):
        self.vk, self.ops, self.n_total = vk, ops, vk.shape[0]

    def rows(self, u1, c0, c1):
        return self.ops.matmul(self.vk[c0:c1], u1, tb=True)


class _TRows:
    """T = (G^T)^+ U1^T (rlra/singlepass.py:135) replicated, sliced by row blocks."""

    def __init__(self, g, ops):
        self.g, self.ops, self.n_total = g, ops, g.shape[0]

    def rows(self, u1, c0, c1):
        t = self.ops.pinv_transpose_apply(self.g, self.ops.transpose(u1))
        out = self.ops.empty(c1 - c0, t.shape[1])
        out.copy_(t[c0:c1])
        return out


def lu_from_projection(A: ShardedMatrix, g_local, vk):
    """rlra/fixedrank.py:136-146 over the row shards: the exact GEPP of G and
    of B^T = V_k U1^T run row-sharded (dist_getrf_: bit-identical to the
    one-GPU kernel, so p and q are the reference's), L = L1 U2^T by row blocks
    (DistLU), U = L2^T.  RLRA_B200_DIST_GEPP=0: G all-gathered and factored
    redundantly on every rank (round 1)."""
    ops = A.ops
    k = g_local.shape[1]
    if DIST_GEPP and A.world > 1 and hasattr(ops, "gepp_state"):
        piv1, piv2, big_l, big_u, _ = _lu_factors_sharded(A, g_local, _BtRows(vk, ops), k)
        return DistLU(piv1, piv2, big_l, big_u, k, A.r0, A.r1, A.m, A.group, ops)
    g = A.gather_rows(g_local)
    piv1, cnt = ops.getrf_(g)
    l1, u1 = ops.lu_extract(g)
    bt = ops.matmul(vk, u1, tb=True)
    piv2, _ = ops.getrf_(bt)
    l2, u2 = ops.lu_extract(bt)
    return _assemble(A, l1, u2, l2, piv1, piv2, k)


# ---------------------------------------------------------------- sharded factorizations of replicated sketches
# Z = A^T W is replicated after its all-reduce (n x l).  Its factorizations run
# on row blocks of Z, one per rank, instead of redundantly on every rank
# (the replicated n x l QR / LU capped the 8-GPU efficiency).
def _row_block(A, rows):
    return row_range(rows, A.world, A.rank)


def _all_gather_rows(A, local, rows):
    """Column-major (rows x w) from the ranks' row blocks (row_range(rows))."""
    w = local.shape[1]
    per = -(-rows // A.world)
    buf = torch.zeros((w, per), dtype=local.dtype, device=local.device)
    if local.shape[0]:
        buf[:, :local.shape[0]].copy_(local.t())
    out = [torch.empty_like(buf) for _ in range(A.world)]
    dist.all_gather(out, buf, group=A.group)
    full = A.ops.empty(rows, w)
    for r in range(A.world):
        a0, a1 = row_range(rows, A.world, r)
        if a1 > a0:
            full[a0:a1, :].copy_(out[r][:, : a1 - a0].t())
    return full


def _block_ok(A, rows, l):
    """Every rank's row block of a rows x l matrix has at least l rows."""
    return A.world > 1 and rows // A.world >= l and row_range(rows, A.world, A.world - 1)[1] - \
        row_range(rows, A.world, A.world - 1)[0] >= l


def sharded_qr_basis(A, z):
    """Orthonormal basis of range(z), z replicated n x l, computed on row
    blocks: CholeskyQR2 with all-reduced l x l Grams (Q_r = Z_r R^{-1}, twice),
    then one all-gather of Q.  When the Cholesky declines (cond(Z) beyond its
    bound -- the decision is identical on every rank, the Gram is replicated),
    TSQR: local Householder QR of each block, the stacked R factors
    all-gathered and factored, Q_r = Q_r,local Q_s[r].  Same range and column
    signs up to +-1 as the Householder Q of the whole z (which no powerlu
    output depends on).  Returns (Q replicated, nonzero-diagonal count or None)."""
    ops = A.ops
    n, l = z.shape
    c0, c1 = _row_block(A, n)
    zr = z[c0:c1]
    if hasattr(ops, "chol_inv") and ops.cholqr_ok(z):
        from .ops import CHOLQR_COND

        # CholeskyQR2, or shifted CholeskyQR3 for sketches wider than the
        # one-CTA Cholesky (ops.scholqr3): all-reduced Grams, local Q_r updates
        wide = ops.cholqr_wide(l)
        steps = [(True, 1e300), (False, 1e7), (False, 2.0)] if wide else [(False, CHOLQR_COND), (False, 2.0)]
        flag = _new_flag(z)
        q = zr
        for i, (shifted, limit) in enumerate(steps):
            g = ops.matmul(q, q, ta=True)
            dist.all_reduce(g.t(), op=dist.ReduceOp.SUM, group=A.group)
            if shifted:
                ops.shift_gram(g, n, flag)
            if i == len(steps) - 1:
                ops.gram_identity_flag(g, flag)
            rinv, flag = ops.chol_inv(g, limit, flag)
            q = ops.matmul(q, rinv)
        if not ops.flag_value(flag):
            return _all_gather_rows(A, q, n), None
    # TSQR
    work = ops.empty(c1 - c0, l)
    work.copy_(zr)
    q_loc, r_loc = ops.qr_qr(work)
    rs = [torch.empty((l, l), dtype=z.dtype, device=z.device) for _ in range(A.world)]
    dist.all_gather(rs, r_loc.contiguous(), group=A.group)  # R_r, row-major
    stacked = ops.empty(A.world * l, l)
    stacked.copy_(torch.cat(rs, 0))
    q_s, r = ops.qr_qr(stacked)
    q_r = ops.matmul(q_loc, q_s[A.rank * l:(A.rank + 1) * l])
    return _all_gather_rows(A, q_r, n), ops.nonzero_diag(r)


def _new_flag(like):
    return torch.zeros(1, dtype=torch.int32, device=like.device)


def sharded_lu_basis(A, z, l):
    """Interior LU basis of a REPLICATED n x l sketch by tournament pivoting
    over row blocks (like tslu_basis_rows for the row-sharded m x l sketch):
    local GEPP of Z_r names l candidates, one all-gather of the world*l x l
    candidates, a redundant GEPP gives U, W_r = Z_r U^{-1}, W all-gathered.
    W = Z U^{-1} with U upper triangular."""
    n = z.shape[0]
    c0, c1 = _row_block(A, n)
    sub = ShardedMatrix(z[c0:c1], n, c0, c1, A.ops, A.group)
    w_r = tslu_basis_rows(sub, z[c0:c1], l)
    return _all_gather_rows(A, w_r, n)


SHARD_REPLICATED = os.environ.get("RLRA_B200_DIST_SHARD_REPL", "1") == "1"  # 0: redundant n x l QR / LU
REPL_TSLU_MIN_ROWS = int(os.environ.get("RLRA_B200_DIST_REPL_TSLU_ROWS", "131072"))

def powerlu(A: ShardedMatrix, k, q_os=10, v=3, seed=0, omega_fn=None):
    """rlra/fixedrank.py:120-133 over a row-sharded A; every rank returns the
    same factors (replicated)."""
    m, n = A.shape
    if k < 1:
        raise ValueError("target rank must be >= 1")
    if q_os < 0:
        raise ValueError("oversampling must be >= 0")
    if k + q_os > min(m, n):
        raise ValueError(f"sketch width {k + q_os} exceeds min{(m, n)}")
    with A.products():
        V, _ = general_power_basis_v(A, k + q_os, v, seed, omega_fn, fast_qr=True)
        vk = V[:, :k]
        g_local = A.matmul(vk)
    return lu_from_projection(A, g_local, vk)


def adaptive_rank(A: ShardedMatrix, eps, b, l, v, seed, omega_fn):
    """rlra/fixedprec.py:57-94 over a row-sharded A (energies all-reduced)."""
    from .fixedprec import scan_energies
    import math

    m, n = A.shape
    if l > min(m, n):
        raise ValueError(f"sketch width {l} exceeds min{(m, n)}")
    with A.products():
        V, _ = general_power_basis_v(A, l, v, seed, omega_fn)
        g_local = A.matmul(V)
    e = A.ops.colsumsq(g_local).clone()
    dist.all_reduce(e, op=dist.ReduceOp.SUM, group=A.group)
    total = math.sqrt(float(A.fro_norm_sq().item())) ** 2
    rank, resid, conv = scan_energies(total, e.cpu().numpy(), eps, b, l)
    return rank, V, g_local, resid, conv


def powerlu_fp(A: ShardedMatrix, eps, b, l, v, seed, omega_fn):
    """rlra/fixedprec.py:152-163 over a row-sharded A: (factors, rank)."""
    rank, V, g_local, resid, conv = adaptive_rank(A, eps, b, l, v, seed, omega_fn)
    if not conv:
        from .fixedprec import AdaptiveOutcome

        raise NotConverged(AdaptiveOutcome(rank, V[:, :rank], g_local[:, :rank], resid, conv))
    # lu_from_projection factors the all-gathered copy, g_local stays intact
    return lu_from_projection(A, g_local[:, :rank], V[:, :rank]), rank


# ---------------------------------------------------------------- single pass
def stream_sketch(A: ShardedMatrix, k, seed, omega_fn, panel=256):
    """rlra/singlepass.py:99-120 over a row-sharded A (each rank streams the
    columns of its own rows A_i, ascending, each column once).

    Per sweep panel J (the single-GPU grouping, singlepass.sweep_width):
      G_J  = A_i(:, J)^T Omega_i   local partial (w x k)
      all-reduce(G_J)              asynchronous: runs while the next panel's
                                   partial product is computed
      H_i += A_i(:, J) G_J         local rows of H
    Returns (G replicated n x k, H_i this rank's rows of the m x k H)."""
    m, n = A.shape
    if not 1 <= k <= min(m, n):
        raise ValueError(f"k={k} outside 1..min{(m, n)}")
    if panel < 1:
        raise ValueError("panel width must be >= 1")
    ops = A.ops
    rows = A.r1 - A.r0
    om = omega_fn(seed, m, k)
    if isinstance(om, torch.Tensor):
        om_i = om[A.r0:A.r1]
    else:
        om_i = ops.upload(np.asfortranarray(om[A.r0:A.r1]))
    oz = hasattr(ops, "sweep_oz") and ops.sweep_oz(m, n, k)
    width = ops.sweep_width(m, panel) if oz else panel
    g = ops.empty(n, k)
    h = ops.zeros(rows, k)
    pending = None  # (j0, w, block, prep, reduced buffer, async handle)

    def finish(item):
        j0, w, block, prep, buf, handle = item
        handle.wait()
        g[j0:j0 + w, :].copy_(buf)
        if rows:
            ops.sweep_products(block, prep, buf, h, ta=False, add=True)  # H_i += A_i(:, J) G_J

    for j0 in range(0, n, width):
        w = min(width, n - j0)
        block = A.local[:, j0:j0 + w]
        prep = ops.sweep_prep(block, oz) if (rows and hasattr(ops, "sweep_prep")) else None
        buf = ops.zeros(w, k)  # contiguous column-major: (k, w) row-major storage
        if rows:
            ops.sweep_products(block, prep, om_i, buf, ta=True, add=False)  # partial G_J
        handle = dist.all_reduce(buf.t(), op=dist.ReduceOp.SUM, group=A.group, async_op=True)
        if pending is not None:
            finish(pending)
        pending = (j0, w, block, prep, buf, handle)
        A.product_count += 1
    if pending is not None:
        finish(pending)
    return g, h


def single_pass_lu(A: ShardedMatrix, k, seed, omega_fn, q_os=0, panel=256):
    """rlra/singlepass.py:123-144 over a row-sharded A; every rank returns the
    same factors.  H is all-gathered for the exact GEPP (p identical to one
    GPU); G, T and their factors are replicated."""
    l = k + q_os
    ops = A.ops
    g, h_local = stream_sketch(A, l, seed, omega_fn, panel)
    if DIST_GEPP and A.world > 1 and hasattr(ops, "gepp_state"):
        piv1, piv2, big_l, big_u, _ = _lu_factors_sharded(A, h_local, _TRows(g, ops), l)
        if q_os:
            big_l, big_u = big_l[:, :k], big_u[:k, :]
        return DistLU(piv1, piv2, big_l, big_u, k, A.r0, A.r1, A.m, A.group, ops)
    h = A.gather_rows(h_local)
    piv1, _ = ops.getrf_(h)
    l1, u1 = ops.lu_extract(h)
    t = ops.pinv_transpose_apply(g, ops.transpose(u1))
    piv2, _ = ops.getrf_(t)
    l2, u2 = ops.lu_extract(t)
    return _assemble(A, l1, u2, l2, piv1, piv2, k, cut=k if q_os else None)


# ---------------------------------------------------------------- drop-in API glue
def _omega(A):
    if A.omega_fn is not None:
        return A.omega_fn
    from . import core

    dev = A.local.device
    return lambda seed, rows, l: core.omega(seed, rows, l, dev)


def shard_rows(a, group=None, device=None, ops=None):
    """This rank's row shard of an m x n matrix (host ndarray or tensor, the
    same full matrix on every rank, or already only this rank's rows with
    `rows_only`): rows row_range(m, world, rank), column-major in HBM."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    m = int(a.shape[0])
    r0, r1 = row_range(m, world, rank)
    if ops is None:
        import torch as _t

        dev = device if device is not None else _t.device("cuda", _t.cuda.current_device())
        ops = CudaOps(dev)
    if isinstance(a, torch.Tensor):
        local = ops.empty(r1 - r0, a.shape[1])
        local.copy_(a[r0:r1])
    else:
        local = ops.upload(np.asfortranarray(np.asarray(a, dtype=np.float64)[r0:r1]))
    return ShardedMatrix(local, m, r0, r1, ops, group)


def api_powerlu(A, k, q_os, v, seed):
    """powerlu(a, k, q_os, v, seed) for a ShardedMatrix (rlra/fixedrank.py:120)."""
    from .fixedrank import LowRankLU

    f = powerlu(A, k, q_os, v, seed, _omega(A))
    return LowRankLU(f.p, f.q, f.full_L(), f.U, f.rank)


def api_adaptive_rank(A, params, seed):
    """adaptive_rank(a, params, seed) (rlra/fixedprec.py:57): G holds this
    rank's rows of A V."""
    from .fixedprec import AdaptiveOutcome

    rank, V, g_local, resid, conv = adaptive_rank(A, params.eps, params.b, params.l, params.v, seed, _omega(A))
    return AdaptiveOutcome(rank, V[:, :rank], g_local[:, :rank], resid, conv)


def api_powerlu_fp(A, params, seed):
    """powerlu_fp(a, params, seed) (rlra/fixedprec.py:152): (LowRankLU,
    AdaptiveOutcome) or NotConverged."""
    from .fixedprec import AdaptiveOutcome
    from .fixedrank import LowRankLU

    rank, V, g_local, resid, conv = adaptive_rank(A, params.eps, params.b, params.l, params.v, seed, _omega(A))
    out = AdaptiveOutcome(rank, V[:, :rank], g_local[:, :rank], resid, conv)
    if not conv:
        raise NotConverged(out)
    f = lu_from_projection(A, g_local[:, :rank], V[:, :rank])
    return LowRankLU(f.p, f.q, f.full_L(), f.U, f.rank), out


def api_general_power_basis_v(A, l, v, seed):
    """general_power_basis_v(a, l, v, seed) (rlra/rangefinder.py:144)."""
    from .rangefinder import RangeBasis

    basis, passes = general_power_basis_v(A, l, v, seed, _omega(A))
    return RangeBasis(basis, passes)


def api_stream_sketch(A, k, seed, panel):
    """stream_sketch(stream, k, seed, panel) (rlra/singlepass.py:99): H holds
    this rank's rows."""
    from .singlepass import SketchPair

    g, h = stream_sketch(A, k, seed, _omega(A), panel)
    return SketchPair(g, h)


def api_single_pass_lu(A, k, seed, q_os, panel):
    """single_pass_lu(stream, k, seed, q_os, panel) (rlra/singlepass.py:123)."""
    from .fixedrank import LowRankLU

    f = single_pass_lu(A, k, seed, _omega(A), q_os=q_os, panel=panel)
    return LowRankLU(f.p, f.q, f.full_L(), f.U, f.rank)
