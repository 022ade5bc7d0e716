"""Rebuild the GEPP golden inputs: small cases are stored in gepp.npz, large
ones are regenerated from their recipe (the same NumPy Generator calls the
reference's rlra.core.gaussian makes, rlra/core.py:33-48)."""

import numpy as np

GAUSSIAN_CASES = [(1, 1), (1, 5), (5, 1), (6, 6), (23, 11), (11, 23), (64, 40),
                  (300, 120), (700, 64), (257, 33)]
TALL_CASES = {"tall_2000x96": (77, 2000, 96), "tall_4100x70": (78, 4100, 70)}


def gaussian(seed, m, n):
    return np.random.default_rng(seed).standard_normal(m * n).reshape((m, n), order="F")


def gepp_input(name, npz):
    if f"{name}/a" in npz:
        return np.asfortranarray(npz[f"{name}/a"])
    if name in TALL_CASES:
        seed, m, n = TALL_CASES[name]
        return gaussian(seed, m, n)
    if name.startswith("rand_"):
        shape, s = name[len("rand_"):].split("_s")
        m, n = (int(x) for x in shape.split("x"))
        return gaussian(1000 * int(s) + m, m, n)
    raise KeyError(name)
