"""Device operands: the reference's accessor protocol (rlra/accessors.py:17-100)
and column-stream protocol (rlra/singlepass.py:27-57) over HBM-resident data.

A ``DeviceMatrix`` holds A column-major in HBM (one upload); ``matmul`` and
``rmatmul`` are one pass over A each (K1/K2: the int8 tensor-core emulation of
csrc/ozaki.cu, or the DMMA GEMM with RLRA_B200_PASS_GEMM=dmma), ``fro_norm`` is
the compensated K2b reduction.  Host ndarrays handed to the drivers are wrapped
in a DeviceMatrix; duck-typed host accessors are adapted so their products feed
the device pipeline (their own products run wherever they run).
"""

from __future__ import annotations

import contextlib
import math
import os

import numpy as np
import torch

from . import ops

DEFAULT_PANEL = 256  # rlra/singlepass.py:19

# Pass-product engine: "oz" = FP64 emulated on the int8 tensor cores
# (csrc/ozaki.cu, DGEMM-level accuracy, ~5x the DMMA pass), "dmma" = native
# FP64 DMMA GEMM (csrc/gemm_tma.cu).
PASS_GEMM = os.environ.get("RLRA_B200_PASS_GEMM", "oz")
OZ_MAX_K = 133144
# residues take nmod bytes per element of A (14 B vs 8 B of float64); operands
# whose residues do not fit in the free HBM (ops.oz_residue_budget; C5 on one
# GPU: 120 GB next to its 68.7 GB A) use block-wise residues (ops.OzBlocked),
# bit-identical to the one-block product
OZ_MAX_RESIDUE_BYTES = None  # None: ops.oz_residue_budget (free memory); RLRA_B200_OZ_MAX_BYTES overrides


_ENGINE = [None]  # per-call override of PASS_GEMM (pass_engine)


@contextlib.contextmanager
def pass_engine(name):
    """Run the pass products of the enclosed calls on `name` ("oz" | "dmma")."""
    prev, _ENGINE[0] = _ENGINE[0], name
    try:
        yield
    finally:
        _ENGINE[0] = prev


def product_session(a):
    """Context in which the pass products of one driver call share the int8
    residues of A (built at the first product, dropped at exit)."""
    fn = getattr(a, "products", None)
    return fn() if fn is not None else contextlib.nullcontext()


class DeviceMatrix:
    """HBM-resident dense operand (rlra/accessors.py:17-37 on device)."""

    is_device_accessor = True

    # Host arrays in pinned memory above this size are uploaded in column
    # chunks on a copy stream; the first product consumes chunks as they land
    # (H2D overlapped with Omega and the first pass -- the e2e path).
    PIPELINE_MIN_BYTES = 256 << 20
    PIPELINE_CHUNKS = 8

    def __init__(self, a, device=None):
        dev = ops.check_device(device)
        self._pending = []  # [(c0, c1, event)] column chunks still in flight
        self._host_keep = None
        if isinstance(a, torch.Tensor):
            if a.dim() != 2:
                raise ValueError(f"expected a 2-d array, got ndim={a.dim()}")
            t = a.to(device=dev, dtype=torch.float64)
            self._a = ops.as_fmat(t)
        else:
            arr = np.asfortranarray(np.asarray(a, dtype=np.float64))
            if arr.ndim != 2:
                raise ValueError(f"expected a 2-d array, got ndim={arr.ndim}")
            host = torch.from_numpy(arr) if arr.size else None
            if host is not None and arr.nbytes >= self.PIPELINE_MIN_BYTES and host.is_pinned():
                self._upload_pipelined(arr, host, dev)
            else:
                self._a = ops.from_numpy(arr, dev)
        self._fro = None
        self._sessions = 0
        self._oz_prep = None

    @contextlib.contextmanager
    def products(self):
        self._sessions += 1
        try:
            yield self
        finally:
            self._sessions -= 1
            if self._sessions == 0:
                self._oz_prep = None

    def _oz_ok(self, k, ncols):
        m, n = self._a.shape
        return (_ENGINE[0] or PASS_GEMM) == "oz" and 0 < k and 0 < ncols <= 4096 and min(m, n) > 0

    def _oz(self):
        """Residues of A for this product session (or a transient one): all
        of A (ops.OzPrep) when they fit next to it, else block-wise
        (ops.OzBlocked: cached blocks + per-product rebuilt blocks)."""
        if self._oz_prep is not None:
            return self._oz_prep
        with ops.label("oz_prep"):
            prep = ops.oz_engine(self.tensor, OZ_MAX_RESIDUE_BYTES)
        if self._sessions > 0:
            self._oz_prep = prep
        return prep

    def _upload_pipelined(self, arr, host, dev):
        m, n = arr.shape
        self._a = ops.fmat(m, n, dev)
        self._host_keep = arr  # the copies read it asynchronously
        copy_stream = torch.cuda.Stream(dev)
        # the destination allocation must be ready before the copy stream writes it
        copy_stream.wait_stream(torch.cuda.current_stream(dev))
        # chunks of whole 256-column blocks: the residues of each chunk are built
        # as it lands (ops.OzPipeline aligns norms and residue tiles to them)
        step = max(256, -(-(-(-n // self.PIPELINE_CHUNKS)) // 256) * 256)
        with torch.cuda.stream(copy_stream):
            for c0 in range(0, n, step):
                c1 = min(n, c0 + step)
                self._a[:, c0:c1].copy_(host[:, c0:c1], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy_stream)
                self._pending.append((c0, c1, ev))
        self._a.record_stream(copy_stream)  # allocator: the copy stream writes this block
        self._copy_stream = copy_stream

    def _finish_upload(self):
        if self._pending:
            st = torch.cuda.current_stream(self.device)
            for _, _, ev in self._pending:
                st.wait_event(ev)
            self._pending = []

    @property
    def shape(self):
        return tuple(self._a.shape)

    @property
    def tensor(self):
        self._finish_upload()
        return self._a

    @property
    def device(self):
        return self._a.device

    def _pipeline(self):
        """Residue builder riding the upload (ops.OzPipeline) when this call's
        later products will take the int8 engine's one-block path."""
        m, n = self._a.shape
        if self._sessions == 0 or self._oz_prep is not None or not self._oz_ok(max(m, n), 1):
            return None
        if max(m, n) > ops.OZ_BLOCK_K or not ops._small_residues(ops.OZ_NMOD * m * n, self.device):
            return None
        return ops.OzPipeline(self._a)

    def _end_pipeline(self, pipe):
        if pipe is not None:
            with ops.label("oz_prep"):
                self._oz_prep = pipe.finish()

    def matmul_with_energies(self, x):
        """(A @ X, column energies sum((A X)[:, j]**2) as a device vector): on
        the int8 engine the energies are reduced inside the product's CRT step
        (rlra/fixedprec.py:71-80 without a second read of G); otherwise the K8
        reduction runs on the product."""
        x = _dev(x, self.device)
        if not self._pending and self._oz_ok(self._a.shape[1], x.shape[1]):
            with ops.label("pass_nn"):
                return self._oz().gemm(x, trans=False, colsq=True)
        y = self.matmul(x)
        return y, ops.colsumsq(y)

    def matmul(self, x):
        """A @ X, one pass over A (rlra/accessors.py:27-28)."""
        x = _dev(x, self.device)
        with ops.label("pass_nn"):
            if self._pending:  # first pass behind the upload: Y = sum_c A_c X_c
                st = torch.cuda.current_stream(self.device)
                y = ops.fmat(self._a.shape[0], x.shape[1], self.device)
                pipe = self._pipeline()
                for i, (c0, c1, ev) in enumerate(self._pending):
                    st.wait_event(ev)
                    ops.gemm(self._a[:, c0:c1], x[c0:c1, :], y, beta=0.0 if i == 0 else 1.0)
                    if pipe is not None:
                        pipe.chunk(c0, c1)
                self._finish_upload()
                self._end_pipeline(pipe)
                return y
            if self._oz_ok(self._a.shape[1], x.shape[1]):
                return self._oz().gemm(x, trans=False)
            return ops.matmul(self._a, x)

    def rmatmul(self, x):
        """A^T @ X, one pass over A (rlra/accessors.py:30-31)."""
        x = _dev(x, self.device)
        with ops.label("pass_tn"):
            if self._pending:  # first pass behind the upload: Z[c] = A_c^T X per chunk
                st = torch.cuda.current_stream(self.device)
                z = ops.fmat(self._a.shape[1], x.shape[1], self.device)
                pipe = self._pipeline()
                for c0, c1, ev in self._pending:
                    st.wait_event(ev)
                    ops.gemm(self._a[:, c0:c1], x, z[c0:c1, :], ta=True)
                    if pipe is not None:
                        pipe.chunk(c0, c1)
                self._finish_upload()
                self._end_pipeline(pipe)
                return z
            if self._oz_ok(self._a.shape[0], x.shape[1]):
                return self._oz().gemm(x, trans=True)
            return ops.matmul(self._a, x, ta=True)

    def fro_norm_sq_device(self):
        """||A||_F^2 as a device scalar (no host sync): inside a product session
        whose residues are built, the by-product of their norms pass (fixed-
        order double-double over the column partials -- no extra read of A);
        otherwise the compensated K2b reduction."""
        self._finish_upload()
        prep = self._oz_prep
        if prep is not None and getattr(prep, "fro2", None) is not None:
            return prep.fro2
        return ops.sumsq(self._a)

    def fro_norm(self):
        """||A||_F (rlra/accessors.py:33-34)."""
        return math.sqrt(float(self.fro_norm_sq_device().item()))

    def to_dense(self):
        self._finish_upload()
        return ops.to_numpy(self._a)


class HostAccessorAdapter:
    """Adapts a duck-typed host accessor (anything with shape/matmul/rmatmul,
    rlra/accessors.py:94-100) to device operands: products are computed by the
    wrapped object and uploaded."""

    is_device_accessor = True

    def __init__(self, inner, device=None):
        self.inner = inner
        self._dev = ops.check_device(device)

    @property
    def shape(self):
        return tuple(self.inner.shape)

    @property
    def device(self):
        return self._dev

    def matmul(self, x):
        return ops.from_numpy(np.asarray(self.inner.matmul(ops.to_numpy(x))), self._dev)

    def rmatmul(self, x):
        return ops.from_numpy(np.asarray(self.inner.rmatmul(ops.to_numpy(x))), self._dev)

    def fro_norm(self):
        return float(self.inner.fro_norm())

    def fro_norm_sq_device(self):
        return torch.tensor([self.fro_norm() ** 2], dtype=torch.float64, device=self._dev)


class InstrumentedAccessor:
    """Counts product invocations (passes) like rlra/accessors.py:67-91."""

    is_device_accessor = True

    def __init__(self, inner):
        self.inner = as_accessor(inner)
        self.product_count = 0

    @property
    def shape(self):
        return self.inner.shape

    @property
    def device(self):
        return self.inner.device

    def products(self):
        return product_session(self.inner)

    def matmul(self, x):
        self.product_count += 1
        return self.inner.matmul(x)

    def rmatmul(self, x):
        self.product_count += 1
        return self.inner.rmatmul(x)

    def matmul_with_energies(self, x):
        self.product_count += 1
        fused = getattr(self.inner, "matmul_with_energies", None)
        if fused is not None:
            return fused(x)
        y = self.inner.matmul(x)
        return y, ops.colsumsq(y)

    def fro_norm(self):
        # a norm query is not a product (rlra/accessors.py:86-88)
        return self.inner.fro_norm()

    def fro_norm_sq_device(self):
        return self.inner.fro_norm_sq_device()

    def to_dense(self):
        return self.inner.to_dense()


def as_accessor(a, device=None):
    """Device analogue of rlra/accessors.py:94-100."""
    if getattr(a, "is_device_accessor", False):
        return a
    if hasattr(a, "matmul") and hasattr(a, "rmatmul") and hasattr(a, "shape"):
        return HostAccessorAdapter(a, device)
    try:
        import scipy.sparse as sp

        if sp.issparse(a):
            return SparseDeviceMatrix(a, device)
    except ImportError:  # pragma: no cover
        pass
    return DeviceMatrix(a, device)


class SparseDeviceMatrix:
    """HBM-resident sparse operand (rlra/accessors.py:40-64, SparseAccessor):
    products never densify A.  Both CSR(A) (for A X) and CSR(A^T) = CSC(A)
    (for A^T X) are kept, int64 indices, so each product is a gather SpMM with
    a fixed per-row summation order (csrc/misc.cu spmm_csr_kernel)."""

    is_device_accessor = True

    def __init__(self, a, device=None):
        import scipy.sparse as sp

        dev = ops.check_device(device)
        self._dev = dev
        csr = sp.csr_matrix(a, dtype=np.float64)
        csr.sum_duplicates()
        csc = sp.csc_matrix(csr)
        self._shape = tuple(int(x) for x in csr.shape)
        up = lambda x, dt: torch.as_tensor(np.ascontiguousarray(x, dtype=dt), device=dev)  # noqa: E731
        self._r = (up(csr.indptr, np.int64), up(csr.indices, np.int64), up(csr.data, np.float64))
        self._c = (up(csc.indptr, np.int64), up(csc.indices, np.int64), up(csc.data, np.float64))
        self._host = csc

    @property
    def shape(self):
        return self._shape

    @property
    def device(self):
        return self._dev

    def _spmm(self, mats, rows, x):
        x = _dev(x, self._dev)
        y = ops.fmat(rows, x.shape[1], self._dev)
        rp, ci, va = mats
        ops._call("rlra_b200_spmm_csr", self._dev, ops.ptr(rp), ops.ptr(ci), ops.ptr(va), rows, ops.ptr(x),
                  ops.ld_of(x), x.shape[1], ops.ptr(y), ops.ld_of(y), ops._stream(self._dev))
        return y

    def matmul(self, x):
        """A @ X, one pass (rlra/accessors.py:50-51)."""
        with ops.label("pass_nn_sparse"):
            return self._spmm(self._r, self._shape[0], x)

    def rmatmul(self, x):
        """A^T @ X, one pass (rlra/accessors.py:53-54)."""
        with ops.label("pass_tn_sparse"):
            return self._spmm(self._c, self._shape[1], x)

    def fro_norm_sq_device(self):
        v = self._r[2]
        return ops.sumsq(v.view(-1, 1)) if v.numel() else torch.zeros(1, dtype=torch.float64, device=self._dev)

    def fro_norm(self):
        """rlra/accessors.py:56-57."""
        return math.sqrt(float(self.fro_norm_sq_device().item()))

    def to_dense(self):
        return np.asarray(self._host.todense(), dtype=np.float64)

    @property
    def sparse(self):
        return self._host


def _dev(x, device):
    if isinstance(x, torch.Tensor):
        if x.device != device:
            x = x.to(device)
        return ops.as_fmat(x.to(torch.float64))
    return ops.from_numpy(x, device)


# ---------------------------------------------------------------- column streams
class _StreamBase:
    """Single-use pull interface (rlra/singlepass.py:27-46)."""

    def __init__(self, shape):
        self.shape = shape
        self.columns_pulled = 0
        self._spent = False

    def panels(self, width=DEFAULT_PANEL):
        if self._spent:
            raise RuntimeError("stream already consumed; columns are single-use")
        if width < 1:
            raise ValueError("panel width must be >= 1")
        self._spent = True
        n = self.shape[1]
        for j0 in range(0, n, width):
            j1 = min(j0 + width, n)
            block = self._panel(j0, j1)
            self.columns_pulled += j1 - j0
            yield j0, block


class DeviceColumnStream(_StreamBase):
    """Streams an HBM-resident matrix by column panels (views, no copies)."""

    def __init__(self, a, device=None):
        self._m = a if isinstance(a, DeviceMatrix) else DeviceMatrix(a, device)
        super().__init__(self._m.shape)

    @property
    def device(self):
        return self._m.device

    def _panel(self, j0, j1):
        return self._m.tensor[:, j0:j1]


from .streams import DenseColumnStream, RlraFileColumnStream  # noqa: E402  (host streams: pinned pipeline)
