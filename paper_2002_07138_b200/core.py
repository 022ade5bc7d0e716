"""Host-side plumbing kept from the reference: the seeded Gaussian stream.

Omega must be bit-identical to the reference's draw (shared-seed comparisons,
rlra/core.py:33-48), so it is produced by the same NumPy PCG64 generator on the
host and uploaded.  ``set_omega_cache(True)`` keeps recent device copies keyed
by (seed, rows, cols, device) -- Omega is a pure function of those -- so
repeated factorizations skip the host draw (bench.py's device-resident `value`
uses it; its e2e number does not).
"""

from __future__ import annotations

from collections import OrderedDict

import numpy as np

from . import ops

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


def omega(seed, m, n, device):
    """Device copy of gaussian(seed, m, n)."""
    key = (int(seed), int(m), int(n), str(device))
    if _cache_on and key in _cache:
        _cache.move_to_end(key)
        return _cache[key]
    om = ops.from_numpy(gaussian(seed, m, n), device)
    if _cache_on:
        _cache[key] = om
        while len(_cache) > _CACHE_MAX:
            _cache.popitem(last=False)
    return om
