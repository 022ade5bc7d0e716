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


PINNED_MIN_BYTES = 1 << 20  # results at least this large come back through pinned buffers


def _host_like(t):
    pin = t.numel() * t.element_size() >= PINNED_MIN_BYTES
    if t.dim() == 1:
        return torch.empty(t.shape, dtype=t.dtype, pin_memory=pin)
    m, n = t.shape
    return torch.empty((n, m), dtype=t.dtype, pin_memory=pin).t()


def to_numpy_many(ts):
    """Download several device tensors (column-major matrices or vectors) with
    asynchronous copies into pinned host buffers and ONE synchronisation;
    returns F-ordered ndarrays viewing those buffers."""
    hosts = []
    for t in ts:
        h = _host_like(t)
        h.copy_(t, non_blocking=True)
        hosts.append(h)
    if ts:
        torch.cuda.current_stream(ts[0].device).synchronize()
    return [h.numpy() for h in hosts]


def to_numpy(t):
    """Download a column-major device matrix as an F-ordered ndarray."""
    return to_numpy_many([t])[0]


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
OZ_HEADER_BYTES = 64  # include/rlra_b200.h RLRA_B200_OZ_HEADER_BYTES
OZ_FRO2_OFFSET = 40  # double ||A||_F^2 in the header


def oz_guard(header, m, n):
    """(ok_nn, ok_tn) from a workspace header (rlra_b200_oz_guard, host only):
    an orientation may take the emulated product only when its error bound is
    within DGEMM's classical bound (csrc/ozaki.cu accuracy note)."""
    import ctypes

    raw = bytes(header.cpu().numpy().tobytes()) if isinstance(header, torch.Tensor) else bytes(header)
    if len(raw) < OZ_HEADER_BYTES:
        raise ValueError("oz header must hold RLRA_B200_OZ_HEADER_BYTES bytes")
    buf = ctypes.create_string_buffer(raw, len(raw))
    ok_nn, ok_tn = ctypes.c_int(0), ctypes.c_int(0)
    _native.call("rlra_b200_oz_guard", ctypes.cast(buf, ctypes.c_void_p), int(m), int(n), ctypes.byref(ok_nn),
                 ctypes.byref(ok_tn))
    return bool(ok_nn.value), bool(ok_tn.value)


def oz_guard_stats(header):
    """Decoded guard header: (max norm, min row norm, min column norm,
    non-finite, integer-valued) -- diagnostics only."""
    h = header.cpu().numpy() if isinstance(header, torch.Tensor) else np.frombuffer(bytes(header), np.uint8)
    mx, mr, mc = h[8:32].view(np.uint64)
    nf, nonint = (int(x) for x in h[32:40].view(np.uint32))
    f = lambda b: float("inf") if b == np.uint64(0xFFFFFFFFFFFFFFFF) else float(np.sqrt(np.array([b]).view(np.float64)[0]))  # noqa: E731
    return f(mx), f(mr), f(mc), bool(nf), not nonint


_SIDE = {}


class _HeaderCopy:
    def __init__(self, buf, ev):
        self.buf, self.ev = buf, ev

    def wait(self):
        self.ev.synchronize()
        return self.buf.clone()


def _header_copy_async(ws, device, nbytes=OZ_HEADER_BYTES):
    """Copy the guard header to pinned host memory on a side stream ordered
    after the work queued so far on the current stream."""
    key = str(device)
    if key not in _SIDE:
        _SIDE[key] = torch.cuda.Stream(device)
    side = _SIDE[key]
    buf = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)  # per copy (the host allocator caches it)
    main = torch.cuda.current_stream(device)
    side.wait_stream(main)
    with torch.cuda.stream(side):
        buf.copy_(ws[:nbytes], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(side)
    ws.record_stream(side)
    return _HeaderCopy(buf, ev)


class OzPrep:
    """Int8 residues of A for the emulated pass products (csrc/ozaki.cu): built
    once per A, they serve both C = A B (trans=False) and C = A^T B.

    guard=True (the product path): the norms and guard statistics are computed
    first and read back (one small device->host transfer on a side stream while
    the residue kernel runs); an orientation the guard rejects (graded rows /
    columns beyond rlra_b200_oz_guard_limit(K), NaN / Inf, extreme exponent
    range, integer-valued A) runs on the FP64 DMMA GEMM instead.  guard=False
    exercises the raw engine (tests)."""

    _resolve_fn = None

    def _resolve(self):
        """Pipelined preps (OzPipeline) read their guard header lazily."""
        if self._resolve_fn is not None:
            fn, self._resolve_fn = self._resolve_fn, None
            fn()

    def __init__(self, a, nmod=None, guard=True):
        m, n = a.shape
        self.a = a
        self.m, self.n = int(m), int(n)
        self.nmod = OZ_NMOD if nmod is None else int(nmod)
        self.device = a.device
        wsb = _native.query("rlra_b200_oz_prep_workspace", self.m, self.n, self.nmod)
        self.ws = torch.empty(max(wsb, 8), dtype=torch.uint8, device=a.device)
        st = _stream(a.device)
        if guard:
            _call("rlra_b200_oz_norms", a.device, ptr(a), ld_of(a), self.m, self.n, self.nmod, ptr(self.ws), wsb, st)
            # the guard header goes to the host on a side stream while the
            # residue kernel (~0.8 ms at C2) already runs on the main stream:
            # the host decision no longer leaves the GPU idle; a rejected
            # orientation only wastes those residues
            host = _header_copy_async(self.ws, a.device)
            _call("rlra_b200_oz_prep_ex", a.device, ptr(a), ld_of(a), self.m, self.n, self.nmod, ptr(self.ws),
                  ptr(self.ws), wsb, st)
            if guard == "lazy":  # read at the first product (tall_prep: issued well before it is needed)
                self.header, self.ok = None, None

                def resolve():
                    self.header = host.wait()
                    self.ok = oz_guard(self.header, self.m, self.n)

                self._resolve_fn = resolve
            else:
                self.header = host.wait()
                self.ok = oz_guard(self.header, self.m, self.n)
        else:
            self.header = None
            self.ok = (True, True)
            _call("rlra_b200_oz_prep", a.device, ptr(a), ld_of(a), self.m, self.n, self.nmod, ptr(self.ws), wsb, st)
        # ||A||_F^2 of the norms pass (header bytes 40..48): device scalar, no extra read of A
        self.fro2 = self.ws[OZ_FRO2_OFFSET:OZ_FRO2_OFFSET + 8].view(torch.float64)

    def gemm(self, b, trans=False, keep_ws=False, out=None, add=False, colsq=False, b_ws=None):
        """C = A B (trans=False, b n x l) or A^T B (trans=True, b m x l); with
        `out`, the product is written into it (add=True: out += A B).
        colsq=True also returns the column energies sum(C[:, j]**2) (device
        vector), reduced inside the product's CRT step -- no second read of C
        (rlra/fixedprec.py:71-80): the result is (C, energies).
        keep_ws=True returns (C, workspace); passing that workspace back as b_ws
        to a product of a prep of the SAME shape with the SAME b and trans skips
        the scales and residues of b (RLRA_B200_OZ_REUSE_B; the single-pass
        sweep multiplies every panel^T by the same Omega)."""
        if colsq and keep_ws:
            raise ValueError("oz gemm: colsq and keep_ws are exclusive")
        k, rows = (self.m, self.n) if trans else (self.n, self.m)
        if b.shape[0] != k:
            raise ValueError(f"oz gemm shape mismatch: A {(self.m, self.n)} trans={trans}, B {tuple(b.shape)}")
        ncols = int(b.shape[1])
        c = fmat(rows, ncols, self.device) if out is None else out
        if tuple(c.shape) != (rows, ncols):
            raise ValueError(f"oz gemm output shape {tuple(c.shape)}, expected {(rows, ncols)}")
        if ncols == 0:
            if colsq:
                return c, torch.zeros(0, dtype=F64, device=self.device)
            return (c, None) if keep_ws else c
        b = as_fmat(b)
        self._resolve()
        if not self.ok[int(bool(trans))]:  # guard: DGEMM-class accuracy needs the native FP64 GEMM
            gemm(self.a, b, c, ta=bool(trans), beta=1.0 if add else 0.0)
            if colsq:
                return c, colsumsq(c)
            return (c, None) if keep_ws else c
        wsb = _native.query("rlra_b200_oz_gemm_workspace", int(trans), self.m, self.n, ncols, self.nmod)
        reuse = b_ws is not None and b_ws.numel() == max(wsb, 8)
        ws = b_ws if reuse else torch.empty(max(wsb, 8), dtype=torch.uint8, device=self.device)
        flags = (OZ_ADD_TO_C if add else 0) | (OZ_COLSQ if colsq else 0) | (OZ_REUSE_B if reuse else 0)
        _call("rlra_b200_oz_gemm_ex", self.device, int(trans), ptr(self.ws), self.m, self.n, self.nmod, ptr(b),
              ld_of(b), ncols, ptr(c), ld_of(c), ptr(ws), wsb, None, flags, _stream(self.device))
        if colsq:
            energies = torch.empty(ncols, dtype=F64, device=self.device)
            _call("rlra_b200_oz_colsq", self.device, int(trans), self.m, self.n, self.nmod, ncols, ptr(ws), wsb,
                  ptr(energies), 0, _stream(self.device))
            return c, energies
        return (c, ws) if keep_ws else c


class OzPipeline:
    """Residues of A built WHILE its column chunks upload (the e2e path,
    device.DeviceMatrix pipelined upload): per chunk the norms partials and the
    residues of its tile columns, with a provisional eA from the first chunk
    (rlra_b200_oz_scale_provisional); after the last chunk the final norms,
    guard statistics and eA.  When the final eA differs from the provisional
    one the residues are rebuilt with it, so the result equals OzPrep's bit
    for bit.  finish() returns the OzPrep."""

    def __init__(self, a, nmod=None):
        self.a = a
        self.m, self.n = int(a.shape[0]), int(a.shape[1])
        self.nmod = OZ_NMOD if nmod is None else int(nmod)
        self.device = a.device
        self.wsb = _native.query("rlra_b200_oz_prep_workspace", self.m, self.n, self.nmod)
        self.ws = torch.empty(max(self.wsb, 8), dtype=torch.uint8, device=a.device)
        self.first = True
        self.rebuilt = False

    def chunk(self, c0, c1):
        a, dev, st = self.a, self.device, _stream(self.device)
        _call("rlra_b200_oz_norms_cols", dev, ptr(a), ld_of(a), self.m, self.n, int(c0), int(c1), self.nmod,
              ptr(self.ws), self.wsb, st)
        if self.first:
            _call("rlra_b200_oz_scale_provisional", dev, self.m, self.n, int(c1), self.nmod, ptr(self.ws), self.wsb,
                  st)
            self.first = False
        _call("rlra_b200_oz_residue_cols", dev, ptr(a), ld_of(a), self.m, self.n, int(c0), int(c1), self.nmod,
              ptr(self.ws), self.wsb, st)

    def finish(self):
        """Final norms / guard statistics / eA queued; the host reads them only
        when the first product needs them (OzPrep._resolve), so the GPU goes on
        with the next step (the interior LU) instead of idling on a sync."""
        a, dev, st = self.a, self.device, _stream(self.device)
        e_final = torch.empty(1, dtype=torch.int32, device=dev)
        _call("rlra_b200_oz_norms_finish", dev, ptr(a), ld_of(a), self.m, self.n, self.nmod, ptr(self.ws), self.wsb,
              ptr(e_final), st)
        hdr = torch.empty(OZ_HEADER_BYTES + 4, dtype=torch.uint8, device=dev)
        hdr[:OZ_HEADER_BYTES].copy_(self.ws[:OZ_HEADER_BYTES])
        hdr[OZ_HEADER_BYTES:].copy_(e_final.view(torch.uint8))
        prep = OzPrep.__new__(OzPrep)
        prep.a, prep.m, prep.n, prep.nmod, prep.device, prep.ws = a, self.m, self.n, self.nmod, dev, self.ws
        prep.fro2 = self.ws[OZ_FRO2_OFFSET:OZ_FRO2_OFFSET + 8].view(torch.float64)
        prep.header, prep.ok = None, None
        pipe = self
        pending = _header_copy_async(hdr, dev, OZ_HEADER_BYTES + 4)  # queued now, read at the first product

        def resolve():
            host = pending.wait()
            e_prov = int(host[:4].view(torch.int32)[0])
            e_fin = int(host[OZ_HEADER_BYTES:].view(torch.int32)[0])
            if e_prov != e_fin:  # the provisional scale did not hold: residues again, with the final one
                pipe.ws[:4].copy_(e_final.view(torch.uint8))
                _call("rlra_b200_oz_prep_ex", dev, ptr(a), ld_of(a), pipe.m, pipe.n, pipe.nmod, ptr(pipe.ws),
                      ptr(pipe.ws), pipe.wsb, _stream(dev))
                host[:4] = host[OZ_HEADER_BYTES:]
                pipe.rebuilt = True
            prep.header = host[:OZ_HEADER_BYTES].clone()
            prep.ok = oz_guard(prep.header, pipe.m, pipe.n)

        prep._resolve_fn = resolve
        return prep


OZ_BLOCK_K = 133120  # largest multiple of 256 inside the exact int32 K range (133144)
OZ_ACCUMULATE, OZ_NO_CRT, OZ_ADD_TO_C, OZ_COLSQ, OZ_REUSE_B = 1, 2, 4, 8, 16  # include/rlra_b200.h


def _split(total, cap):
    """[(s0, s1)] cutting `total` into equal pieces of at most `cap`, each a
    multiple of 256 except the last."""
    nb = max(1, -(-total // cap))
    step = -(-(-(-total // nb)) // 256) * 256
    return [(s, min(total, s + step)) for s in range(0, total, step)]


class OzBlocked:
    """Pass products of an A whose residues do not fit next to it, or whose K
    exceeds the exact int32 range (C5: 262144 x 32768 needs 120 GB of
    residues next to its 68.7 GB).  A is cut into row x column blocks that
    share ONE scale eA (norms over the whole A) and every product one
    per-column scale eB of the whole B, so K-split products accumulate their
    residues exactly (RLRA_B200_OZ_ACCUMULATE) and the result is bit-identical
    to OzPrep's.  Residues of as many blocks as the memory budget allows are
    kept for the product session; the others are rebuilt per product in one
    scratch workspace (8 B read + nmod B written per element)."""

    last_stats = None  # of the most recent engine (bench.py's C5 sub-record reports it)

    def __init__(self, a, nmod=None, block_bytes=None, cache_bytes=None, row_cap=OZ_BLOCK_K,
                 col_cap=OZ_BLOCK_K, guard=True):
        m, n = a.shape
        self.a = a
        self.m, self.n = int(m), int(n)
        self.nmod = OZ_NMOD if nmod is None else int(nmod)
        self.device = a.device
        dev = a.device
        wsb = _native.query("rlra_b200_oz_scale_workspace", self.m, self.n)
        ws = torch.empty(max(wsb, 8), dtype=torch.uint8, device=dev)
        self.e_a = torch.empty(1, dtype=torch.int32, device=dev)
        _call("rlra_b200_oz_scale", dev, ptr(a), ld_of(a), self.m, self.n, self.nmod, ptr(self.e_a), ptr(ws), wsb,
              _stream(dev))
        self.header = ws[:OZ_HEADER_BYTES].cpu() if guard else None
        self.ok = oz_guard(self.header, self.m, self.n) if guard else (True, True)
        self.fro2 = ws[OZ_FRO2_OFFSET:OZ_FRO2_OFFSET + 8].view(torch.float64).clone()
        del ws
        if block_bytes is None:
            block_bytes = int(os.environ.get("RLRA_B200_OZ_BLOCK_BYTES", str(16 << 30)))
        # full-width row blocks when n allows (long K for the NN product, K
        # split -- exact accumulation -- only in the TN product)
        self.cols = _split(self.n, min(int(col_cap), OZ_BLOCK_K))
        wb = self.cols[0][1] - self.cols[0][0]
        hcap = max(256, min(int(row_cap), OZ_BLOCK_K, (block_bytes // (self.nmod * wb)) // 256 * 256))
        self.rows = _split(self.m, hcap)
        self.blocks = [(i, j) for i in range(len(self.rows)) for j in range(len(self.cols))]
        size = lambda ij: _native.query("rlra_b200_oz_prep_workspace", self.rows[ij[0]][1] - self.rows[ij[0]][0],
                                        self.cols[ij[1]][1] - self.cols[ij[1]][0], self.nmod)
        self.block_ws = {ij: size(ij) for ij in self.blocks}
        biggest = max(self.block_ws.values())
        if not any(self.ok):  # every product goes to the DMMA GEMM: no residues at all
            self.blocks = []
        total = sum(self.block_ws.values())
        if cache_bytes is None:
            free, _ = torch.cuda.mem_get_info(dev)
            free += torch.cuda.memory_reserved(dev) - torch.cuda.memory_allocated(dev)  # allocator cache
            cache_bytes = free - OZ_RESERVE_BYTES
        self.scratch = None
        if self.blocks and total > cache_bytes:
            # the scratch block first, while the largest contiguous range is free
            self.scratch = torch.empty(biggest, dtype=torch.uint8, device=dev)
            cache_bytes -= biggest
        self.cache = {}
        used = 0
        for ij in self.blocks:
            if used + self.block_ws[ij] <= cache_bytes:
                try:
                    self.cache[ij] = self._build(ij, None)
                except torch.OutOfMemoryError:  # fragmented allocator: rebuild the rest per product
                    if self.scratch is None:
                        self.scratch = torch.empty(biggest, dtype=torch.uint8, device=dev)
                    break
                used += self.block_ws[ij]
        if self.scratch is not None and len(self.cache) == len(self.blocks):
            self.scratch = None
        self.rebuilt = len(self.blocks) - len(self.cache)
        OzBlocked.last_stats = {"blocks": len(self.blocks), "cached": len(self.cache), "rebuilt_per_product": self.rebuilt,
                                "row_blocks": len(self.rows), "col_blocks": len(self.cols)}

    def _build(self, ij, into):
        (r0, r1), (c0, c1) = self.rows[ij[0]], self.cols[ij[1]]
        wsb = self.block_ws[ij]
        ws = into if into is not None else torch.empty(max(wsb, 8), dtype=torch.uint8, device=self.device)
        a = self.a
        _call("rlra_b200_oz_prep_ex", self.device, ptr(a) + (r0 + c0 * ld_of(a)) * 8, ld_of(a), r1 - r0, c1 - c0,
              self.nmod, ptr(self.e_a), ptr(ws), wsb, _stream(self.device))
        return ws

    def _prep(self, ij):
        ws = self.cache.get(ij)
        return ws if ws is not None else self._build(ij, self.scratch)

    def gemm(self, b, trans=False, colsq=False):
        """C = A B (trans=False, b n x l) or A^T B (trans=True, b m x l);
        colsq=True: (C, column energies of C), reduced in the CRT steps."""
        k, rows = (self.m, self.n) if trans else (self.n, self.m)
        if b.shape[0] != k:
            raise ValueError(f"oz gemm shape mismatch: A {(self.m, self.n)} trans={trans}, B {tuple(b.shape)}")
        ncols = int(b.shape[1])
        c = fmat(rows, ncols, self.device)
        if ncols == 0:
            return (c, torch.zeros(0, dtype=F64, device=self.device)) if colsq else c
        b = as_fmat(b)
        if not self.ok[int(bool(trans))]:  # guard (OzPrep): the native FP64 GEMM
            gemm(self.a, b, c, ta=bool(trans))
            return (c, colsumsq(c)) if colsq else c
        energies = torch.empty(ncols, dtype=F64, device=self.device) if colsq else None
        dev, st = self.device, _stream(self.device)
        cp = int(_native.load().rlra_b200_oz_cols_pad(ncols))
        e_b = torch.empty(cp, dtype=torch.int32, device=dev)
        _call("rlra_b200_oz_bscale", dev, ptr(b), ld_of(b), k, ncols, self.nmod, ptr(e_b), st)
        wsb = max(_native.query("rlra_b200_oz_gemm_workspace", int(trans), r1 - r0, c1 - c0, ncols, self.nmod)
                  for (r0, r1) in self.rows for (c0, c1) in self.cols)
        ws = torch.empty(max(wsb, 8), dtype=torch.uint8, device=dev)
        # output blocks (outer) x K blocks (inner, accumulated exactly)
        outer, inner = (self.cols, self.rows) if trans else (self.rows, self.cols)
        for o, (o0, o1) in enumerate(outer):
            for q, (k0, k1) in enumerate(inner):
                ij = (q, o) if trans else (o, q)
                (r0, r1), (c0, c1) = self.rows[ij[0]], self.cols[ij[1]]
                last = q + 1 == len(inner)
                flags = (OZ_ACCUMULATE if q > 0 else 0) | (0 if last else OZ_NO_CRT) | (OZ_COLSQ if colsq and last else 0)
                _call("rlra_b200_oz_gemm_ex", dev, int(trans), ptr(self._prep(ij)), r1 - r0, c1 - c0, self.nmod,
                      ptr(b) + k0 * 8, ld_of(b), ncols, ptr(c) + o0 * 8, ld_of(c), ptr(ws), wsb, ptr(e_b), flags, st)
                if colsq and last:  # this output row block's share of every column's energy
                    _call("rlra_b200_oz_colsq", dev, int(trans), r1 - r0, c1 - c0, self.nmod, ncols, ptr(ws), wsb,
                          ptr(energies), 1 if o > 0 else 0, st)
        return (c, energies) if colsq else c


OZ_RESERVE_BYTES = int(os.environ.get("RLRA_B200_OZ_RESERVE_BYTES", str(12 << 30)))


def oz_residue_budget(device):
    """Bytes the residues of one operand may take: RLRA_B200_OZ_MAX_BYTES, else
    the device's free memory (allocator cache included) minus a reserve for the
    sketches and workspaces (C5 on one GPU: 120 GB of residues next to its
    68.7 GB A do not fit -> block-wise; a C5 row shard at 2+ GPUs does)."""
    env = os.environ.get("RLRA_B200_OZ_MAX_BYTES")
    if env:
        return int(env)
    free, _ = torch.cuda.mem_get_info(device)
    free += torch.cuda.memory_reserved(device) - torch.cuda.memory_allocated(device)
    return max(0, free - OZ_RESERVE_BYTES)


_TOTAL_MEM = {}


def _small_residues(nbytes, device):
    """Residues under an eighth of the device memory need no free-memory query
    (the query -- cudaMemGetInfo plus the allocator's statistics -- costs
    ~0.3 ms of host time at the start of every call, GPU idle)."""
    if os.environ.get("RLRA_B200_OZ_MAX_BYTES"):
        return False
    key = str(device)
    if key not in _TOTAL_MEM:
        _TOTAL_MEM[key] = torch.cuda.get_device_properties(device).total_memory
    return nbytes <= _TOTAL_MEM[key] // 8


def oz_engine(a, max_residue_bytes=None):
    """OzPrep when the residues of all of A fit (and K is in range), else OzBlocked."""
    m, n = a.shape
    if max_residue_bytes is None and max(m, n) <= OZ_BLOCK_K and _small_residues(OZ_NMOD * m * n, a.device):
        return OzPrep(a)
    if max_residue_bytes is None:
        max_residue_bytes = oz_residue_budget(a.device)
    if max(m, n) <= OZ_BLOCK_K and OZ_NMOD * m * n <= max_residue_bytes:
        return OzPrep(a)
    return OzBlocked(a)


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


def tn_tall(x, y):
    """x^T y for tall x, y (n x l, n x w): the int8 engine (residues of x, TN
    product with B = y) when x is large, else the DMMA GEMM."""
    n, l = x.shape
    if (os.environ.get("RLRA_B200_PASS_GEMM", "oz") == "oz" and n * l >= CHOLQR_OZ_MIN_ELEMS
            and n <= OZ_BLOCK_K and y.shape[1] <= 4096):
        return OzPrep(x).gemm(y, trans=True)
    return matmul(x, y, ta=True)


def _diag_blocks(l, cap):
    nb = max(1, -(-l // cap))
    step = -(-l // nb)
    return [(j, min(l, j + step)) for j in range(0, l, step)]


def chol_inv_blocked(g, out, flag, cond_limit):
    """out = chol(g)^{-1} (upper) for any l; g (full symmetric) is consumed.

    l <= chol_inv_max_l: the one-CTA kernel.  Wider: diagonal blocks by the
    one-CTA kernel (R_JJ^{-1}, condition bound inside the block), block rows
    R_J,rest = R_JJ^{-T} G_J,rest and trailing updates G_rest -= R_J,rest^T
    R_J,rest on the DMMA GEMM, then R^{-1} assembled block column by block
    column (Rinv_0J = -Rinv_00 R_0J Rinv_JJ) and the condition bound across
    blocks on its diagonal (|Rinv_ii| = 1 / |R_ii|)."""
    l = g.shape[0]
    cap = cholqr_max_l()
    if l <= cap:
        return chol_inv(g, out, flag, cond_limit)
    dev = g.device
    blocks = _diag_blocks(l, cap)
    r = fmat(l, l, dev, zero=True)  # off-diagonal blocks of R
    out.zero_()
    for j0, j1 in blocks:
        gjj = fmat(j1 - j0, j1 - j0, dev)
        gjj.copy_(g[j0:j1, j0:j1])
        chol_inv(gjj, out[j0:j1, j0:j1], flag, cond_limit)
        if j1 < l:
            gemm(out[j0:j1, j0:j1], g[j0:j1, j1:], r[j0:j1, j1:], ta=True)
            gemm(r[j0:j1, j1:], r[j0:j1, j1:], g[j1:, j1:], ta=True, alpha=-1.0, beta=1.0)
    for j0, j1 in blocks[1:]:
        t = matmul(out[:j0, :j0], r[:j0, j0:j1])
        gemm(t, out[j0:j1, j0:j1], out[:j0, j0:j1], alpha=-1.0)
    _call("rlra_b200_diag_ratio_flag", dev, ptr(out), ld_of(out), l, float(cond_limit), ptr(flag), _stream(dev))
    return out


SCHOL_C = 11.0 * 2.0 ** -53  # shift constant of shifted CholeskyQR (Fukaya et al. 2020)
CHOLQR_OZ_MIN_ELEMS = int(os.environ.get("RLRA_B200_CHOLQR_OZ_MIN", str(1 << 24)))


# Tall x small factor products (rlra/fixedrank.py:144-146 L = L1 U2^T and
# (U1 V^T)^T = V U1^T; rlra/kernels.py:95-96 Q (R^-T M)): 2 rows k^2 flops with a
# tall operand whose rows are evenly scaled (unit-lower L1, orthonormal V / Q) --
# on the int8 engine 2-3x the DMMA rate once the product is large enough.  The
# residues are issued EARLY (before the GEPP that precedes the product), so the
# guard header has long arrived when the product reads it: no host wait.
FACTOR_OZ_MIN_WORK = float(os.environ.get("RLRA_B200_FACTOR_OZ_MIN_WORK", "5e9"))   # rows * k * ncols
FACTOR_OZ_MAX_ELEMS = float(os.environ.get("RLRA_B200_FACTOR_OZ_MAX_ELEMS", "6e7"))  # rows * k (workspace 28 B each)


def tall_prep(a, ncols):
    """Residues of the tall operand `a` (rows x k) for a later a @ s with s
    k x ncols (tall_times), or None when the FP64 DMMA GEMM is the better engine
    (small products; C5's 262144 x 512 factor, whose 4 GB of residue workspace
    would come out of the memory the block-wise pass engine budgets)."""
    rows, k = a.shape
    if (os.environ.get("RLRA_B200_PASS_GEMM", "oz") != "oz" or rows * k * ncols < FACTOR_OZ_MIN_WORK
            or rows * k > FACTOR_OZ_MAX_ELEMS or k > OZ_BLOCK_K or ncols > 4096 or ncols < 1):
        return None
    with label("factor_prep"):
        return OzPrep(as_fmat(a), guard="lazy")


def tall_times(a, s, prep=None, ts=False):
    """a @ s (ts=False) or a @ s^T (ts=True), a tall and s small; `prep` =
    tall_prep(a, .) issued earlier, else the DMMA GEMM."""
    if prep is not None:
        with label("factor_oz"):
            return prep.gemm(transpose(s) if ts else s, trans=False)
    return matmul(a, s, tb=ts)


def _tall_products(z):
    """(gram, times) for a tall sketch z: Z^T Z and Z R.  Large sketches (C3-C5
    final bases, C4's pinv) take the int8 tensor-core engine -- ONE residue set
    of z serves both products (TN with B = z, NN with B = R) -- under its
    dynamic-range guard; small ones the DMMA GEMM."""
    n, l = z.shape
    if (os.environ.get("RLRA_B200_PASS_GEMM", "oz") == "oz" and n * l >= CHOLQR_OZ_MIN_ELEMS
            and n <= OZ_BLOCK_K and l <= 4096):
        prep = OzPrep(z)
        return (lambda: prep.gemm(z, trans=True)), (lambda r: prep.gemm(r, trans=False))
    return (lambda: matmul(z, z, ta=True)), (lambda r: matmul(z, r))
NO_COND_LIMIT = 1e300


def scholqr3(z):
    """Orthonormal basis of range(z) by shifted CholeskyQR3 (csrc/cholqr.cu
    notes): step 1 factors Z^T Z + s I, s = 11 (n l + l (l + 1)) u ||Z||_F^2,
    which succeeds for cond(Z) up to ~u^-1 and leaves cond(Q1) ~ 1e4; steps 2
    and 3 are CholeskyQR2 on Q1 with the usual condition bounds.  All six
    products are DMMA GEMMs, the factorizations blocked Choleskys (any l).
    The device flag is raised when step 2 or 3 declines, or when z has an
    exactly zero column (the structural rank collapse the reference's
    Householder R reports as an exact zero diagonal, rlra/rangefinder.py:55-64):
    the caller then redoes the basis on the Householder path."""
    n, l = z.shape
    dev = z.device
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    with label("scholqr3"):
        # exactly zero column -> flag (diag_ratio_flag sees a zero diagonal of Z^T Z)
        q = z
        for step, limit in enumerate((NO_COND_LIMIT, 1e7, 2.0)):
            with label("scholqr3_prep"):
                gram, times = _tall_products(q)
            with label("scholqr3_gram"):
                g = gram()
            if step == 0:
                _call("rlra_b200_diag_ratio_flag", dev, ptr(g), ld_of(g), l, NO_COND_LIMIT, ptr(flag), _stream(dev))
                _call("rlra_b200_chol_shift_diag", dev, ptr(g), ld_of(g), l,
                      SCHOL_C * (n * l + l * (l + 1)), _stream(dev))
            if step == 2:
                gram_identity_flag(g, flag)
            rinv = fmat(l, l, dev)
            with label("scholqr3_chol"):
                chol_inv_blocked(g, rinv, flag, limit)
            with label("scholqr3_q"):
                q = times(rinv)
    return q, flag


def cholqr2(z):
    """Orthonormal basis of range(z) by CholeskyQR2 (csrc/cholqr.cu) and a device
    int32 flag that is 1 when the Cholesky declined (rank collapse or cond(z)
    beyond the bound); z is left intact for the Householder fallback."""
    n, l = z.shape
    dev = z.device
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    rinv = fmat(l, l, dev)
    with label("cholqr2"):
        gram, times = _tall_products(z)
        g = gram()
        chol_inv_blocked(g, rinv, flag, CHOLQR_COND)
        q1 = times(rinv)
        gram, times = _tall_products(q1)
        g2 = gram()
        gram_identity_flag(g2, flag)  # cond(Z) beyond ~u^-1/2 whatever the diagonal ratio said
        chol_inv_blocked(g2, rinv, flag, 2.0)
        q = times(rinv)
    return q, flag


GRAM_IDENTITY_TOL = 0.1


def gram_identity_flag(g, flag, tol=GRAM_IDENTITY_TOL):
    _call("rlra_b200_gram_identity_flag", g.device, ptr(g), ld_of(g), g.shape[0], float(tol), ptr(flag),
          _stream(g.device))


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


def trsm_un_(r, x):
    """x <- R^{-1} x in place, R upper triangular (rlra/fixedrank.py:113)."""
    l = r.shape[0]
    ncols = x.shape[1]
    wsb = _native.query("rlra_b200_trsm_workspace", l, ncols)
    ws = torch.empty(max(wsb, 8), dtype=torch.uint8, device=x.device)
    _call("rlra_b200_trsm_un", x.device, ptr(r), ld_of(r), l, ptr(x), ld_of(x), ncols, ptr(ws), wsb,
          _stream(x.device))
    return x


def apply_inv_row_perm(p, x):
    """out[p[i], :] = x[i, :] (rlra/core.py:103-109)."""
    m, n = x.shape
    out = fmat(m, n, x.device)
    pinv = torch.empty(max(int(m), 1), dtype=I64, device=x.device)
    _call("rlra_b200_apply_inv_row_perm", x.device, ptr(p), m, n, ptr(x), ld_of(x), ptr(pinv), ptr(out),
          ld_of(out), _stream(x.device))
    return out


def svd_jacobi(a):
    """a (m x l, m >= l) = U diag(s) V^T by one-sided Jacobi (csrc/svd.cu);
    s nonincreasing.  Returns (U m x l, s (l,), V l x l, sweeps device int)."""
    m, l = a.shape
    dev = a.device
    u, v = fmat(m, l, dev), fmat(l, l, dev)
    s = torch.empty(max(int(l), 1), dtype=F64, device=dev)[: int(l)]
    sweeps = torch.zeros(1, dtype=torch.int32, device=dev)
    wsb = _native.query("rlra_b200_svd_jacobi_workspace", m, l)
    ws = torch.empty(max(wsb, 8), dtype=torch.uint8, device=dev)
    _call("rlra_b200_svd_jacobi", dev, ptr(a), ld_of(a), m, l, ptr(u), ld_of(u), ptr(s), ptr(v), ld_of(v),
          ptr(sweeps), ptr(ws), wsb, _stream(dev))
    return u, s, v, sweeps


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
