"""Thin typed wrappers over the C ABI on torch device tensors.

Matrices are torch float64 CUDA tensors of shape (m, n) with column-major
strides (1, ld) -- the reference's canonical layout (rlra/core.py:25-30).
Every op enqueues on torch's current stream of the tensor's device; torch is
used only for device memory, streams and views (plumbing), never for math.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _native
from .errors import NativeUnavailable

F64 = torch.float64
I64 = torch.int64


class _Profiler:
    """Optional CUDA-event timing of every C-ABI call (bench.py breakdown and
    the live roofline of the pass GEMMs).  Off by default: zero overhead."""

    def __init__(self):
        self.on = False
        self.records = []  # (label, start_event, end_event)
        self.label = None

    def call(self, name, args, dev):
        if not self.on:
            return _native.call(name, *args)
        st = torch.cuda.current_stream(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        rc = _native.call(name, *args)
        e1.record(st)
        self.records.append((self.label or name, e0, e1))
        return rc

    def summary(self):
        torch.cuda.synchronize()
        out = {}
        for lab, e0, e1 in self.records:
            ms = e0.elapsed_time(e1)
            tot, cnt = out.get(lab, (0.0, 0))
            out[lab] = (tot + ms, cnt + 1)
        return out


PROF = _Profiler()


class label:
    """Tag the C-ABI calls issued inside the block (profiling only)."""

    def __init__(self, name):
        self.name = name

    def __enter__(self):
        self.prev, PROF.label = PROF.label, self.name

    def __exit__(self, *exc):
        PROF.label = self.prev


def _call(name, dev, *args):
    return PROF.call(name, args, dev)


def _stream(dev):
    return ctypes_ptr(torch.cuda.current_stream(dev).cuda_stream)


def ctypes_ptr(x):
    return int(x) if x is not None else None


def check_device(dev=None):
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device visible; the B200 path has no CPU fallback")
    _native.load()
    return torch.device("cuda", torch.cuda.current_device() if dev is None else dev)


# ---------------------------------------------------------------- layout helpers
def fmat(m, n, device, zero=False):
    """Empty (or zeroed) column-major m x n float64 device matrix, ld = max(m, 1)."""
    ld = max(int(m), 1)
    buf = (torch.zeros if zero else torch.empty)((max(int(n), 1), ld), dtype=F64, device=device)
    return buf.t()[: int(m), : int(n)]


def ld_of(t):
    """Leading dimension of a column-major (m, n) view; validates the layout."""
    if t.dtype != F64:
        raise TypeError(f"expected float64, got {t.dtype}")
    m, n = t.shape
    s0, s1 = t.stride()
    if (m > 1 and s0 != 1) or (n > 1 and s1 < max(m, 1)):
        raise ValueError(f"tensor is not column-major (shape {tuple(t.shape)}, strides {t.stride()})")
    return max(s1, m, 1) if n > 1 else max(m, 1)


def as_fmat(t):
    """Column-major view of t (copy only if needed)."""
    try:
        ld_of(t)
        return t
    except ValueError:
        out = fmat(t.shape[0], t.shape[1], t.device)
        out.copy_(t)
        return out


def from_numpy(a, device):
    """Upload a host matrix as a column-major device matrix."""
    a = np.asfortranarray(np.asarray(a, dtype=np.float64))
    if a.ndim != 2:
        raise ValueError(f"expected a 2-d array, got ndim={a.ndim}")
    out = fmat(a.shape[0], a.shape[1], device)
    if a.size:
        out.copy_(torch.from_numpy(a), non_blocking=False)
    return out


def to_numpy(t):
    """Download a column-major device matrix as an F-ordered ndarray."""
    if t.dim() == 1:
        return t.cpu().numpy()
    m, n = t.shape
    host = torch.empty((n, m), dtype=t.dtype).t()
    host.copy_(t)
    return host.numpy()


def ptr(t):
    return t.data_ptr() if t is not None else None


# ---------------------------------------------------------------- kernels
def gemm(a, b, c, *, ta=False, tb=False, alpha=1.0, beta=0.0):
    """c = alpha op(a) op(b) + beta c on the DMMA pipe (K1/K2/K5)."""
    m, n = c.shape
    k = a.shape[0] if ta else a.shape[1]
    if (b.shape[1] if tb else b.shape[0]) != k or (a.shape[1] if ta else a.shape[0]) != m or (
        b.shape[0] if tb else b.shape[1]
    ) != n:
        raise ValueError(f"gemm shape mismatch: op(a) {tuple(a.shape)} ta={ta}, op(b) {tuple(b.shape)} tb={tb}, c {tuple(c.shape)}")
    wsb = _native.query("rlra_b200_gemm_workspace", m, n, k)
    ws = torch.empty(max(wsb, 8), dtype=torch.uint8, device=c.device) if wsb else None
    _call("rlra_b200_dgemm", c.device, int(ta), int(tb), m, n, k, float(alpha), ptr(a), ld_of(a),
                 ptr(b), ld_of(b), float(beta), ptr(c), ld_of(c), ptr(ws), wsb,
                 _stream(c.device))
    return c


OZ_NMOD = int(os.environ.get("RLRA_B200_OZ_NMOD", "14"))


class OzPrep:
    """Int8 residues of A for the emulated pass products (csrc/ozaki.cu): built
    once per A, they serve both C = A B (trans=False) and C = A^T B."""

    def __init__(self, a, nmod=None):
        m, n = a.shape
        self.m, self.n = int(m), int(n)
        self.nmod = OZ_NMOD if nmod is None else int(nmod)
        self.device = a.device
        wsb = _native.query("rlra_b200_oz_prep_workspace", self.m, self.n, self.nmod)
        self.ws = torch.empty(max(wsb, 8), dtype=torch.uint8, device=a.device)
        _call("rlra_b200_oz_prep", a.device, ptr(a), ld_of(a), self.m, self.n, self.nmod, ptr(self.ws), wsb,
              _stream(a.device))

    def gemm(self, b, trans=False, keep_ws=False):
        """C = A B (trans=False, b n x l) or A^T B (trans=True, b m x l)."""
        k, rows = (self.m, self.n) if trans else (self.n, self.m)
        if b.shape[0] != k:
            raise ValueError(f"oz gemm shape mismatch: A {(self.m, self.n)} trans={trans}, B {tuple(b.shape)}")
        ncols = int(b.shape[1])
        c = fmat(rows, ncols, self.device)
        if ncols == 0:
            return (c, None) if keep_ws else c
        b = as_fmat(b)
        wsb = _native.query("rlra_b200_oz_gemm_workspace", int(trans), self.m, self.n, ncols, self.nmod)
        ws = torch.empty(max(wsb, 8), dtype=torch.uint8, device=self.device)
        _call("rlra_b200_oz_gemm", self.device, int(trans), ptr(self.ws), self.m, self.n, self.nmod, ptr(b),
              ld_of(b), ncols, ptr(c), ld_of(c), ptr(ws), wsb, _stream(self.device))
        return (c, ws) if keep_ws else c


def matmul(a, b, *, ta=False, tb=False):
    m = a.shape[1] if ta else a.shape[0]
    n = b.shape[0] if tb else b.shape[1]
    c = fmat(m, n, a.device)
    return gemm(a, b, c, ta=ta, tb=tb)


def iota(m, device):
    p = torch.empty(max(int(m), 1), dtype=I64, device=device)[: int(m)]
    if m:
        _call("rlra_b200_iota", device, ptr(p), int(m), _stream(device))
    return p


def getrf_(a, piv=None):
    """In-place packed GEPP of a (bit-exact with rlra/_lu_cython.pyx:14-55).

    Returns (piv, nonzero_diag_count_device_tensor)."""
    m, n = a.shape
    if piv is None:
        piv = iota(m, a.device)
    cnt = torch.zeros(1, dtype=I64, device=a.device)
    wsb = _native.query("rlra_b200_getrf_workspace", m, n)
    ws = torch.empty(max(wsb, 8), dtype=torch.uint8, device=a.device)
    _call("rlra_b200_getrf", a.device, ptr(a), ld_of(a), m, n, ptr(piv), ptr(cnt), ptr(ws), wsb,
                 _stream(a.device))
    return piv, cnt


def lu_basis(lu, piv, k=None):
    """W = P^T L of a packed LU (rlra/rangefinder.py:73-77)."""
    m, n = lu.shape
    k = min(m, n) if k is None else k
    w = fmat(m, k, lu.device)
    pinv = torch.empty(max(m, 1), dtype=I64, device=lu.device)
    _call("rlra_b200_lu_basis", lu.device, ptr(lu), ld_of(lu), m, k, ptr(piv), ptr(pinv), ptr(w),
                 ld_of(w), _stream(lu.device))
    return w


def lu_extract(lu, want_l=True, want_u=True):
    m, n = lu.shape
    r = min(m, n)
    l = fmat(m, r, lu.device) if want_l else None
    u = fmat(r, n, lu.device) if want_u else None
    _call("rlra_b200_lu_extract", lu.device, ptr(lu), ld_of(lu), m, n, ptr(l),
                 ld_of(l) if l is not None else 1, ptr(u), ld_of(u) if u is not None else 1,
                 _stream(lu.device))
    return l, u


def count_nonzero_diag(a, r=None):
    r = min(a.shape) if r is None else r
    cnt = torch.zeros(1, dtype=I64, device=a.device)
    _call("rlra_b200_count_nonzero_diag", a.device, ptr(a), ld_of(a), r, ptr(cnt), _stream(a.device))
    return cnt


CHOLQR_COND = 2e6  # first-pass bound on max R_ii / min R_ii (CholeskyQR2 needs cond < ~u^-1/2)


def cholqr_max_l():
    return _native.query("rlra_b200_chol_inv_max_l")


def chol_inv(g, out, flag, cond_limit):
    """out = chol(g)^{-1} (upper); flag[0] = 1 when g is not numerically SPD."""
    l = g.shape[0]
    _call("rlra_b200_chol_inv", g.device, ptr(g), ld_of(g), l, ptr(out), ld_of(out), ptr(flag), float(cond_limit),
          _stream(g.device))
    return out


def cholqr2(z):
    """Orthonormal basis of range(z) by CholeskyQR2 (csrc/cholqr.cu) and a device
    int32 flag that is 1 when the Cholesky declined (rank collapse or cond(z)
    beyond the bound); z is left intact for the Householder fallback."""
    n, l = z.shape
    dev = z.device
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    rinv = fmat(l, l, dev)
    with label("cholqr2"):
        g = matmul(z, z, ta=True)
        chol_inv(g, rinv, flag, CHOLQR_COND)
        q1 = matmul(z, rinv)
        g2 = matmul(q1, q1, ta=True)
        chol_inv(g2, rinv, flag, 2.0)
        q = matmul(q1, rinv)
    return q, flag


class QR:
    """geqrf in place + workspace kept for orgqr (rlra/kernels.py:57-61)."""

    def __init__(self, a):
        m, n = a.shape
        if m < n:
            raise ValueError(f"need a tall matrix, got {(m, n)}")
        self.a = a
        self.tau = torch.empty(max(n, 1), dtype=F64, device=a.device)
        self.wsb = _native.query("rlra_b200_geqrf_workspace", m, n)
        self.ws = torch.empty(max(self.wsb, 8), dtype=torch.uint8, device=a.device)
        _call("rlra_b200_geqrf", a.device, ptr(a), ld_of(a), m, n, ptr(self.tau), ptr(self.ws),
                     self.wsb, _stream(a.device))

    def q(self):
        m, n = self.a.shape
        q = fmat(m, n, self.a.device)
        _call("rlra_b200_orgqr", self.a.device, ptr(self.a), ld_of(self.a), m, n, ptr(q), ld_of(q),
                     ptr(self.ws), self.wsb, _stream(self.a.device))
        return q

    def r_view(self):
        n = self.a.shape[1]
        return self.a[:n, :n]


def trsm_rt_(r, x):
    """x <- R^{-T} x in place, R upper triangular (rlra/kernels.py:95)."""
    l = r.shape[0]
    ncols = x.shape[1]
    wsb = _native.query("rlra_b200_trsm_workspace", l, ncols)
    ws = torch.empty(max(wsb, 8), dtype=torch.uint8, device=x.device)
    _call("rlra_b200_trsm_rt", x.device, ptr(r), ld_of(r), l, ptr(x), ld_of(x), ncols, ptr(ws), wsb,
                 _stream(x.device))
    return x


def diag_absmin(a):
    out = torch.empty(1, dtype=F64, device=a.device)
    _call("rlra_b200_diag_absmin", a.device, ptr(a), ld_of(a), min(a.shape), ptr(out), _stream(a.device))
    return out


def sumsq(a):
    """Compensated ||a||_F^2 as a device scalar tensor."""
    m, n = a.shape
    out = torch.zeros(1, dtype=F64, device=a.device)
    wsb = _native.query("rlra_b200_sumsq_workspace", m, n)
    ws = torch.empty(max(wsb, 8), dtype=torch.uint8, device=a.device)
    _call("rlra_b200_sumsq", a.device, ptr(a), ld_of(a), m, n, ptr(out), ptr(ws), wsb, _stream(a.device))
    return out


def colsumsq(a):
    m, n = a.shape
    out = torch.empty(max(n, 1), dtype=F64, device=a.device)[:n]
    _call("rlra_b200_colsumsq", a.device, ptr(a), ld_of(a), m, n, ptr(out), _stream(a.device))
    return out


def transpose(a):
    m, n = a.shape
    out = fmat(n, m, a.device)
    _call("rlra_b200_transpose", a.device, ptr(a), ld_of(a), m, n, ptr(out), ld_of(out), _stream(a.device))
    return out
