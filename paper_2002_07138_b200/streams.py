"""Out-of-core column streams for the single-pass LU.

The reference streams host panels one at a time (rlra/singlepass.py:27-96):
``RlraFileColumnStream`` seeks and reads each panel of a column-major ``.rlm``
file (rlra/fileio.py:14-46), ``DenseColumnStream`` slices an in-memory array.
Here every host-side stream feeds HBM through ONE pipeline:

  reader thread   file / ndarray --(pread | memcpy)--> pinned slot i % R
  copy stream     pinned slot --(async H2D)--> device slot i % R, event copied[i]
  compute stream  waits copied[i], runs panel i's products (K1/K2), event done[i]

with R slots, so the read of panel i+2, the upload of panel i+1 and the
products of panel i overlap.  A pinned slot is refilled only after its upload
completed, a device slot only after the products that consumed it completed.
The matrix never has to fit in HBM (or in host memory, for files): the memory
held is R panels on each side.  Panels arrive in ascending column order, like
the reference, so the sketch accumulation order is unchanged.
"""

from __future__ import annotations

import os
import struct
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

from . import ops

RLRA_MAGIC = b"RLRA"  # rlra/fileio.py:14-15
RLRA_HEADER_BYTES = 4 + 8 + 8
PIPELINE_SLOTS = 3
IO_THREADS = int(os.environ.get("RLRA_B200_IO_THREADS", "8"))  # parallel preads / copies per panel
_POOL = None


def _pool():
    global _POOL
    if _POOL is None:
        _POOL = ThreadPoolExecutor(max_workers=max(1, IO_THREADS), thread_name_prefix="rlra-b200-io")
    return _POOL


def _split_cols(j0, j1, parts):
    step = max(1, -(-(j1 - j0) // parts))
    return [(c, min(j1, c + step)) for c in range(j0, j1, step)]


# ---------------------------------------------------------------- .rlm container
def write_rlra(path, a):
    """rlra/fileio.py:18-25: magic, <u64 rows, <u64 cols, column-major <f8."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError("only 2-d matrices can be stored")
    with open(path, "wb") as fh:
        fh.write(RLRA_MAGIC)
        fh.write(struct.pack("<QQ", a.shape[0], a.shape[1]))
        fh.write(np.asfortranarray(a).tobytes(order="F"))


def read_rlra_header(path):
    """rlra/fileio.py:28-38: (rows, cols) after validating magic and size."""
    with open(path, "rb") as fh:
        head = fh.read(RLRA_HEADER_BYTES)
        if len(head) < RLRA_HEADER_BYTES or head[:4] != RLRA_MAGIC:
            raise IOError(f"{path}: not an RLRA matrix file")
        m, n = struct.unpack("<QQ", head[4:])
        fh.seek(0, 2)
        if fh.tell() != RLRA_HEADER_BYTES + 8 * m * n:
            raise IOError(f"{path}: size does not match declared {m}x{n}")
    return int(m), int(n)


def read_rlra(path):
    """rlra/fileio.py:41-46 (host helper; the product path streams instead)."""
    m, n = read_rlra_header(path)
    with open(path, "rb") as fh:
        fh.seek(RLRA_HEADER_BYTES)
        flat = np.fromfile(fh, dtype="<f8", count=m * n)
    return flat.reshape((m, n), order="F")


# ---------------------------------------------------------------- pipeline
class _Slot:
    def __init__(self, m, width, device):
        self.host = torch.empty((width, m), dtype=torch.float64, pin_memory=True)  # column-major m x width
        self.dev = torch.empty((width, m), dtype=torch.float64, device=device)
        self.uploaded = None  # event: H2D from `host` finished (host slot reusable)
        self.consumed = None  # event: products that read `dev` finished (device slot reusable)


def pipelined_panels(shape, width, fill, device, slots=PIPELINE_SLOTS):
    """Yield (j0, device panel m x w) for every column panel, ascending.

    fill(j0, j1, out) writes columns [j0, j1) into the F-ordered float64
    ndarray `out` (m x (j1 - j0), a view of pinned memory); it runs on a
    background thread (file reads and memcpy release the GIL)."""
    m, n = shape
    if n == 0:
        return
    starts = list(range(0, n, width))
    ring = [_Slot(m, width, device) for _ in range(min(slots, len(starts)))]
    R = len(ring)
    filled = [threading.Event() for _ in starts]
    upload_issued = [threading.Event() for _ in starts]
    errors = []
    stop = threading.Event()

    def reader():
        try:
            for i, j0 in enumerate(starts):
                if stop.is_set():
                    return
                s = ring[i % R]
                if i >= R:  # the previous occupant's H2D must be issued, then complete
                    upload_issued[i - R].wait()
                    if stop.is_set():
                        return
                    s.uploaded.synchronize()
                j1 = min(n, j0 + width)
                out = s.host[: j1 - j0].numpy().T  # F-ordered m x w view
                fill(j0, j1, out)
                filled[i].set()
        except BaseException as e:  # surfaced on the consumer side
            errors.append(e)
            for ev in filled:
                ev.set()

    th = threading.Thread(target=reader, name="rlra-b200-panel-reader", daemon=True)
    th.start()
    copy_stream = torch.cuda.Stream(device)
    compute = torch.cuda.current_stream(device)
    issued = 0

    def issue(i):
        s = ring[i % R]
        filled[i].wait()
        if errors:
            raise errors[0]
        j1 = min(n, starts[i] + width)
        w = j1 - starts[i]
        with torch.cuda.stream(copy_stream):
            if s.consumed is not None:
                copy_stream.wait_event(s.consumed)
            s.dev[:w].copy_(s.host[:w], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy_stream)
        s.uploaded = ev
        upload_issued[i].set()

    try:
        for i, j0 in enumerate(starts):
            if issued == i:
                issue(i)  # waits for the read of panel i
                issued += 1
            # prefetch uploads of panels already read (never block on a read here)
            while issued < len(starts) and issued <= i + R - 1 and filled[issued].is_set():
                issue(issued)
                issued += 1
            s = ring[i % R]
            compute.wait_event(s.uploaded)
            w = min(n, j0 + width) - j0
            yield j0, s.dev[:w].t()
            ev = torch.cuda.Event()
            ev.record(compute)
            s.consumed = ev
    finally:
        stop.set()
        for ev in filled + upload_issued:
            ev.set()
        th.join()
        for s in ring:  # the allocator must not recycle slots still in use on either stream
            s.dev.record_stream(copy_stream)


class _HostStreamBase:
    """Single-use pull interface (rlra/singlepass.py:27-46) over host data,
    delivering device panels through the pinned pipeline."""

    def __init__(self, shape, device=None):
        self.shape = tuple(int(x) for x in shape)
        self.columns_pulled = 0
        self._spent = False
        self._device = device

    @property
    def device(self):
        return ops.check_device(self._device)

    def panels(self, width=256):
        if self._spent:
            raise RuntimeError("stream already consumed; columns are single-use")
        if width < 1:
            raise ValueError("panel width must be >= 1")
        self._spent = True
        for j0, block in pipelined_panels(self.shape, width, self._fill, self.device):
            self.columns_pulled += block.shape[1]
            yield j0, block


class DenseColumnStream(_HostStreamBase):
    """Streams an in-memory HOST matrix (rlra/singlepass.py:49-57) through the
    pinned pipeline (memcpy of each panel, async upload, overlapped)."""

    def __init__(self, a, device=None):
        self._a = np.asfortranarray(np.asarray(a, dtype=np.float64))
        if self._a.ndim != 2:
            raise ValueError(f"expected a 2-d array, got ndim={self._a.ndim}")
        super().__init__(self._a.shape, device)

    def _fill(self, j0, j1, out):
        def cp(c0, c1):
            np.copyto(out[:, c0 - j0:c1 - j0], self._a[:, c0:c1])

        list(_pool().map(lambda r: cp(*r), _split_cols(j0, j1, IO_THREADS)))


class RlraFileColumnStream(_HostStreamBase):
    """Streams a column-major ``.rlm`` file without loading it whole
    (rlra/singlepass.py:60-74): each panel is a contiguous byte range, read
    by IO_THREADS parallel preads straight into pinned memory, then uploaded
    asynchronously."""

    def __init__(self, path, device=None):
        self._path = os.fspath(path)
        super().__init__(read_rlra_header(self._path), device)

    def _fill(self, j0, j1, out):
        m = self.shape[0]
        buf = memoryview(out.T.reshape(-1)).cast("B")  # out is F-ordered: its bytes are contiguous
        fd = os.open(self._path, os.O_RDONLY)

        def rd(c0, c1):  # columns [c0, c1): one contiguous byte range of file and buffer
            lo, hi = 8 * m * (c0 - j0), 8 * m * (c1 - j0)
            got = lo
            while got < hi:
                r = os.preadv(fd, [buf[got:hi]], RLRA_HEADER_BYTES + 8 * m * j0 + got)
                if r <= 0:
                    break
                got += r
            return got == hi

        try:
            ok = all(_pool().map(lambda r: rd(*r), _split_cols(j0, j1, IO_THREADS)))
        finally:
            os.close(fd)
        if not ok:
            raise IOError(f"{self._path}: truncated column data")
        if np.little_endian is False:  # pragma: no cover - the format is little-endian
            out.byteswap(inplace=True)
