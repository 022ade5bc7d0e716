"""Synthetic workloads C1-C5 (BASELINE.json ``configs``; SURVEY.md §8(d) and
Appendix A recipes).  Host-side input generation for tests and bench.py — not
part of the factorization path.

C1 is exactly ``rlra.matgen.gen_decay("custom", 2000, 2000, seed=1, sigma)``
(rlra/matgen.py:36-58).  C2-C5 are ``A = X diag(sigma) Y^T + noise N(0,1)``
with X, Y QR-orthonormalised seeded Gaussians drawn from ONE default_rng
stream in the order X, Y, noise (noise filled column-major), as the survey's
recipe states.  The reference measured its numbers on
these recipes, so the seeds are fixed here.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def _gaussian_from(rng, m, n):
    # rlra/core.py:46-48 — the F-order fill order is part of the contract
    return rng.standard_normal(m * n).reshape((m, n), order="F")


@dataclass(frozen=True)
class Workload:
    name: str
    m: int
    n: int
    k: int
    q_os: int
    v: int
    seed: int = 0  # driver seed for Omega
    kind: str = "powerlu"  # powerlu | powerlu_fp | single_pass
    eps: float = 0.0
    b: int = 0


def gen_c1():
    """C1: 2000x2000 log-uniform decay 1 -> 1e-4 (seed 1)."""
    sigma = 10.0 ** (-4.0 * np.arange(2000) / 1999)
    rng = np.random.default_rng(1)
    u, _ = np.linalg.qr(_gaussian_from(rng, 2000, 2000))
    v, _ = np.linalg.qr(_gaussian_from(rng, 2000, 2000))
    return np.asfortranarray((u * sigma) @ v.T)


def gen_lowrank_plus_noise(m, n, r, sigma, noise, seed, col_chunk=4096):
    """A = X diag(sigma) Y^T + noise * N(0,1); X, Y, noise from one stream.

    The noise is drawn in column blocks: gaussian_from fills column-major, so
    consecutive blocks are exactly the columns of the single full draw (same
    bits), without a second m x n temporary (C5 would need 206 GB)."""
    rng = np.random.default_rng(seed)
    x, _ = np.linalg.qr(_gaussian_from(rng, m, r))
    y, _ = np.linalg.qr(_gaussian_from(rng, n, r))
    a = np.asfortranarray((x * sigma) @ y.T)
    del x, y
    if noise:
        for c0 in range(0, n, col_chunk):
            c1 = min(n, c0 + col_chunk)
            a[:, c0:c1] += noise * _gaussian_from(rng, m, c1 - c0)
    return a


def gen_c2(m=20000, n=10000):
    """C2: rank-400 i^-2 spectrum + 1e-8 noise (seed 2)."""
    return gen_lowrank_plus_noise(m, n, 400, 1.0 / np.arange(1, 401) ** 2, 1e-8, 2)


def gen_c3(n=16384):
    """C3: width-1024 exp(-i/60) spectrum, no noise (seed 3)."""
    return gen_lowrank_plus_noise(n, n, 1024, np.exp(-np.arange(1, 1025) / 60.0), 0.0, 3)


def gen_c4(n=50000):
    """C4: rank-300 i^-1.5 spectrum + 1e-6 noise (seed 4)."""
    return gen_lowrank_plus_noise(n, n, 300, np.arange(1, 301) ** -1.5, 1e-6, 4)


def gen_c5(m=262144, n=32768):
    """C5: width-640 log-uniform 1 -> 1e-8 spectrum + 1e-10 noise (seed 5)."""
    return gen_lowrank_plus_noise(m, n, 640, 10.0 ** (-8.0 * np.arange(640) / 639), 1e-10, 5)


WORKLOADS = {
    "C1": Workload("C1", 2000, 2000, 50, 10, 3),
    "C2": Workload("C2", 20000, 10000, 200, 20, 4),
    "C3": Workload("C3", 16384, 16384, 0, 0, 3, kind="powerlu_fp", eps=1e-6, b=64),
    "C4": Workload("C4", 50000, 50000, 360, 360, 1, kind="single_pass"),
    "C5": Workload("C5", 262144, 32768, 512, 32, 4),
}


def powerlu_flops(m, n, k, l, v):
    """Algorithmic flops of one powerlu.

    Passes 2mn[(v-1)l + k]; GEPP a x b = ab^2 - b^3/3; Householder QR with
    explicit Q of a x b = 4ab^2 - 4b^3/3; assembly GEMMs 2nk^2 + 2mk^2.
    """
    gepp = lambda a, b: a * b * b - b ** 3 / 3.0
    qr = lambda a, b: 4.0 * a * b * b - 4.0 * b ** 3 / 3.0
    passes = 2.0 * m * n * ((v - 1) * l + k)
    fact = qr(n, l) + gepp(m, k) + gepp(n, k) + 2.0 * n * k * k + 2.0 * m * k * k
    if v % 2:
        h = (v - 1) // 2
        fact += h * gepp(m, l) + (h - 1) * gepp(n, l)
    elif v >= 4:
        h = (v - 2) // 2
        fact += h * (gepp(m, l) + gepp(n, l))
    return passes, fact


def single_pass_flops(m, n, l):
    """Algorithmic flops of one single_pass_lu of sketch width l (SURVEY.md
    Appendix B): sweep 4mnl; GEPP(m x l of H) + QR(n x l of G) + 2nl^2 (T = Q X)
    + GEPP(n x l of T) + 2ml^2 (L = L1 U2^T) + l^3 (TRSM)."""
    gepp = lambda a, b: a * b * b - b ** 3 / 3.0
    qr = lambda a, b: 4.0 * a * b * b - 4.0 * b ** 3 / 3.0
    sweep = 4.0 * m * n * l
    fact = gepp(m, l) + qr(n, l) + 2.0 * n * l * l + gepp(n, l) + 2.0 * m * l * l + float(l) ** 3
    return sweep, fact


def powerlu_fp_flops(m, n, l, v, rank):
    """Algorithmic flops of one powerlu_fp: v passes of
    width l (the G pass uses the full l) + 2mn for ||A||_F^2; interior LUs and
    the final QR as in powerlu; the assembly at the chosen rank."""
    gepp = lambda a, b: a * b * b - b ** 3 / 3.0
    qr = lambda a, b: 4.0 * a * b * b - 4.0 * b ** 3 / 3.0
    passes = 2.0 * m * n * v * l + 2.0 * m * n
    fact = qr(n, l) + gepp(m, rank) + gepp(n, rank) + 2.0 * n * rank * rank + 2.0 * m * rank * rank
    if v % 2:
        h = (v - 1) // 2
        fact += h * gepp(m, l) + (h - 1) * gepp(n, l)
    elif v >= 4:
        h = (v - 2) // 2
        fact += h * (gepp(m, l) + gepp(n, l))
    return passes, fact


# ---------------------------------------------------------------- device builds
def gen_device(name, device):
    """Build config `name`'s A directly in HBM (column-major torch tensor).

    Same recipe and random streams as the host generators: X and Y come from
    the seeded NumPy stream and NumPy's QR on the host; the m x n noise is the
    continuation of that same stream drawn by the bit-exact device generator;
    A = (X diag(sigma)) Y^T is formed by the DMMA GEMM.  Equal to the host
    build up to the GEMM's rounding (~1e-16 relative) -- the input generator
    for C3-C5, whose host builds take minutes (C5: 68.7 GB)."""
    import torch

    from . import core, ops

    spec = {
        "C2": (20000, 10000, 400, 1.0 / np.arange(1, 401) ** 2, 1e-8, 2),
        "C3": (16384, 16384, 1024, np.exp(-np.arange(1, 1025) / 60.0), 0.0, 3),
        "C4": (50000, 50000, 300, np.arange(1, 301) ** -1.5, 1e-6, 4),
        "C5": (262144, 32768, 640, 10.0 ** (-8.0 * np.arange(640) / 639), 1e-10, 5),
    }[name]
    m, n, r, sigma, noise, seed = spec
    rng = np.random.default_rng(seed)
    x, _ = np.linalg.qr(_gaussian_from(rng, m, r))
    y, _ = np.linalg.qr(_gaussian_from(rng, n, r))
    xs = ops.from_numpy(np.asfortranarray(x * sigma), device)
    del x
    yd = ops.from_numpy(y, device)
    del y
    a = ops.fmat(m, n, device)
    ops.gemm(xs, yd, a, tb=True)
    del xs, yd
    if noise:
        st = rng.bit_generator.state["state"]
        flat = core.device_gaussian_flat(None, m * n, device, pcg_state=(int(st["state"]), int(st["inc"])))
        if flat is None:
            raise RuntimeError("device generator unavailable for the noise term")
        a.add_(flat.view(n, m).t(), alpha=noise)
        del flat
    torch.cuda.synchronize(device)
    return a
