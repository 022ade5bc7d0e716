"""The seeded Gaussian test matrix Omega (rlra/core.py:33-48).

Omega must be bit-identical to the reference's draw (shared-seed comparisons,
prefix property).  It is generated ON THE DEVICE by librlra_b200's PCG64 +
ziggurat replay of NumPy's ``Generator.standard_normal`` (csrc/rng.cu): the
128-bit PCG64 seed state comes from NumPy itself, the ziggurat tables are read
from the installed NumPy (paper_2002_07138_b200/ziggurat.py), and the rare
tail draws (~1 in 3900) are finished with the host libm ``log1p`` so every
bit matches.  If the constants cannot be validated, or the device pass reports
a failure, the draw falls back to NumPy on the host (Omega is an input, not
part of the factorization arithmetic).

``set_omega_cache(True)`` additionally keeps recent device copies keyed by
(seed, rows, cols, device) -- Omega is a pure function of those.  bench.py's
device-resident `value` uses it; its e2e number does not.
"""

from __future__ import annotations

from collections import OrderedDict

import math

import numpy as np
import torch

from . import _native, ops, ziggurat

_cache: "OrderedDict[tuple, object]" = OrderedDict()
_cache_on = False
_CACHE_MAX = 4


def set_omega_cache(enabled: bool):
    global _cache_on
    _cache_on = bool(enabled)
    if not _cache_on:
        _cache.clear()


def gaussian(seed, m, n):
    """rlra/core.py:33-48: default_rng(seed).standard_normal(m*n) in F order."""
    if m < 1 or n < 1:
        raise ValueError("gaussian needs m, n >= 1")
    return gaussian_from(np.random.default_rng(seed), m, n)


def gaussian_from(rng, m, n):
    """rlra/core.py:46-48."""
    return rng.standard_normal(m * n).reshape((m, n), order="F")


_device_rng = True
_tables = {}


def set_device_rng(enabled: bool):
    """Use the device generator (default) or NumPy on the host for Omega."""
    global _device_rng
    _device_rng = bool(enabled)


def _device_tables(device):
    key = str(device)
    if key not in _tables:
        ki, wi, fi = ziggurat.tables()
        _tables[key] = (torch.from_numpy(ki.view(np.int64)).to(device),
                        torch.from_numpy(wi).to(device), torch.from_numpy(fi).to(device))
    return _tables[key]


def _resolve_tails(words, nbits=16):
    """Host finish of the tail draws (rlra/core.py -> NumPy random_standard_normal
    idx == 0 branch) with libm log1p, as NumPy does: (len, value) per start.

    words: uint64[k, nbits+1] = the start word and the words after it."""
    r_inv, r = ziggurat.ZIGGURAT_NOR_INV_R, ziggurat.ZIGGURAT_NOR_R
    k = words.shape[0]
    lens = np.full(k, -3, dtype=np.int32)
    vals = np.zeros(k)
    for i in range(k):
        w = words[i]
        neg = (int(w[0]) >> 17) & 1  # (rabs >> 8) & 1 with rabs = (u >> 9) & (2^52 - 1)
        j = 1
        while j + 1 <= nbits:
            u1 = (int(w[j]) >> 11) * (1.0 / 9007199254740992.0)
            u2 = (int(w[j + 1]) >> 11) * (1.0 / 9007199254740992.0)
            xx = -r_inv * math.log1p(-u1)
            yy = -math.log1p(-u2)
            j += 2
            if yy + yy > xx * xx:
                lens[i] = j
                vals[i] = -(r + xx) if neg else r + xx
                break
    return lens, vals


_CHUNK = 1 << 28  # normals per device pass (workspace ~20 B per stream word)


def device_gaussian_flat(seed, count, device, pcg_state=None, out=None):
    """gaussian(seed, count, 1).ravel() generated on the device (None if the
    device generator is unavailable or reports a failure).  ``pcg_state`` =
    (state, inc) continues an existing NumPy PCG64 stream instead.  Counts
    beyond 2^28 are produced in chunks, each continuing the PCG64 stream at the
    word where the previous chunk stopped (NumPy PCG64.advance)."""
    if not _device_rng or not ziggurat.validated():
        return None
    state, inc = pcg_state if pcg_state is not None else ziggurat.pcg64_state(seed)
    if out is None:
        out = torch.empty(max(count, 1), dtype=torch.float64, device=device)
    done = 0
    while done < count:
        n = min(_CHUNK, count - done)
        used = _device_gaussian_chunk(state, inc, n, device, out[done:done + n])
        if used is None:
            return None
        done += n
        if done < count:
            bg = np.random.PCG64()
            st = bg.state
            st["state"] = {"state": state, "inc": inc}
            st["has_uint32"], st["uinteger"] = 0, 0
            bg.state = st
            bg.advance(used)
            s2 = bg.state["state"]
            state, inc = int(s2["state"]), int(s2["inc"])
    return out[:count]


def _device_gaussian_chunk(state, inc, count, device, out):
    """One device pass: `count` normals from PCG64 (state, inc) into `out`;
    returns the number of 64-bit words consumed, or None on failure."""
    lib = _native.load()
    ki, wi, fi = _device_tables(device)
    m64 = (1 << 64) - 1
    wsb = int(lib.rlra_b200_normal_workspace(count))
    ws = torch.empty(wsb, dtype=torch.uint8, device=device)
    st = torch.cuda.current_stream(device).cuda_stream
    _native.call("rlra_b200_normal_begin", state >> 64, state & m64, inc >> 64, inc & m64, count,
                 ki.data_ptr(), wi.data_ptr(), fi.data_ptr(), ws.data_ptr(), wsb, st)
    import ctypes

    pu, pt, pn = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    _native.call("rlra_b200_normal_views", count, ws.data_ptr(), ctypes.byref(pu), ctypes.byref(pt),
                 ctypes.byref(pn))
    base = ws.data_ptr()
    T = int(lib.rlra_b200_normal_stream_words(count))
    cap = int(lib.rlra_b200_normal_tail_cap(count))
    u = ws[pu.value - base: pu.value - base + 8 * T].view(torch.int64)
    tpos = ws[pt.value - base: pt.value - base + 8 * cap].view(torch.int64)
    ntail = int(ws[pn.value - base: pn.value - base + 8].view(torch.int64).item())
    if ntail > cap:
        return None
    nb = 16
    if ntail:
        pos = tpos[:ntail]
        idx = (pos.unsqueeze(1) + torch.arange(nb + 1, device=device).unsqueeze(0)).clamp_(max=T - 1)
        words = u[idx].cpu().numpy().view(np.uint64)
        lens, vals = _resolve_tails(words, nb)
        lens[(pos + nb >= T).cpu().numpy()] = -3  # stream end: words were clamped
        tl = torch.from_numpy(lens).to(device)
        tv = torch.from_numpy(vals).to(device)
        tp = pos
    else:
        tl = torch.zeros(1, dtype=torch.int32, device=device)
        tv = torch.zeros(1, dtype=torch.float64, device=device)
        tp = torch.zeros(1, dtype=torch.int64, device=device)
    status = torch.zeros(3, dtype=torch.int64, device=device)
    _native.call("rlra_b200_normal_finish", count, tp.data_ptr(), tl.data_ptr(), tv.data_ptr(), ntail,
                 out.data_ptr(), status.data_ptr(), ws.data_ptr(), wsb, st)
    produced, flags, used = status.cpu().tolist()
    if produced < count or flags:
        return None
    return used


def omega(seed, m, n, device):
    """Device copy of gaussian(seed, m, n) (column-major m x n)."""
    key = (int(seed), int(m), int(n), str(device))
    if _cache_on and key in _cache:
        _cache.move_to_end(key)
        return _cache[key]
    flat = device_gaussian_flat(seed, int(m) * int(n), device)
    if flat is not None:
        om = flat.view(int(n), int(m)).t()  # F-order fill == column-major storage
    else:
        om = ops.from_numpy(gaussian(seed, m, n), device)
    if _cache_on:
        _cache[key] = om
        while len(_cache) > _CACHE_MAX:
            _cache.popitem(last=False)
    return om
