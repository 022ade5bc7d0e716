"""Generate the golden vectors in tests/golden/ from the REFERENCE itself.

Run in the build container (where /root/reference exists), after
``oracle/build_ref.sh`` has installed the unmodified reference into
oracle/_ref:

    python tests/golden/make_golden.py

It imports ``rlra`` (compiled backend) from oracle/_ref and records inputs and
outputs of the hot-path calls on small seeded cases, plus scalar summaries
(rel_err, rank, sha256 of p/q) of the C1 and C2 configs.  The fixtures are
committed; the GPU box never needs /root/reference.  Cases mirror the
reference's own tests (pkg/tests/test_kernels.py, test_backend.py,
test_fixedrank.py, test_fixedprec.py, test_singlepass.py) where those pin the
path.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(REPO, "oracle", "_ref"))
sys.path.insert(0, REPO)
os.environ["RLRA_BACKEND"] = "compiled"

import rlra  # noqa: E402  (the reference, unmodified)
from rlra import core, fixedprec, fixedrank, kernels, matgen, singlepass  # noqa: E402

from paper_2002_07138_b200 import configs  # noqa: E402

assert rlra.BACKEND == "compiled"


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def sha_f64(a):
    """Digest of the column-major float64 bytes (bit-exact comparison)."""
    return hashlib.sha256(np.asfortranarray(a, dtype=np.float64).tobytes(order="F")).hexdigest()


GAUSSIAN_CASES = [(1, 1), (1, 5), (5, 1), (6, 6), (23, 11), (11, 23), (64, 40),
                  (300, 120), (700, 64), (257, 33)]
TALL_CASES = {"tall_2000x96": (77, 2000, 96), "tall_4100x70": (78, 4100, 70)}


def gepp_cases():
    """Inputs for the native kernel seam plu_inplace (rlra/backend.py:32)."""
    cases = {}
    # frozen 2x2 (pkg/tests/test_kernels.py:8-12)
    cases["frozen2x2"] = np.array([[0.0, 1.0], [2.0, 3.0]])
    # tie-break: first maximum wins (pkg/tests/test_backend.py:53-59)
    cases["tie"] = np.array([[1.0, 5.0], [2.0, 6.0], [-2.0, 7.0]])
    # random shapes (pkg/tests/test_backend.py:30-35, test_kernels.py:15-26)
    for (m, n) in GAUSSIAN_CASES:  # input = core.gaussian(1000 * seed + m, m, n)
        for seed in range(2):
            cases[f"rand_{m}x{n}_s{seed}"] = core.gaussian(1000 * seed + m, m, n)
    rng = np.random.default_rng(3)
    col = rng.standard_normal((12, 1))
    # degenerate inputs (pkg/tests/test_backend.py:38-50)
    cases["dupcols"] = np.hstack([col, col, rng.standard_normal((12, 3))])
    cases["zeros"] = np.zeros((8, 5))
    cases["zerorows"] = np.vstack([rng.standard_normal((3, 6)), np.zeros((7, 6))])
    cases["zeroleading"] = np.hstack([np.zeros((9, 2)), rng.standard_normal((9, 4))])
    # duplicated direction -> exactly zero pivot (pkg/tests/test_kernels.py:34-41)
    rng = np.random.default_rng(4)
    col = rng.standard_normal((10, 1))
    cases["dup2x"] = np.hstack([col, 2.0 * col, rng.standard_normal((10, 2))])
    # integer-valued exact rank 5 with many exact ties (pkg/tests/test_cli.py:76-89)
    rng = np.random.default_rng(0)
    picker = np.zeros((60, 5))
    picker[np.arange(60), rng.integers(0, 5, 60)] = 1.0
    cases["int_rank5"] = picker @ rng.integers(1, 9, size=(5, 40)).astype(np.float64)
    # wide-ish panel crossing shapes for the blocked device kernel
    for name, (seed, m, n) in TALL_CASES.items():  # input = core.gaussian(seed, m, n)
        cases[name] = core.gaussian(seed, m, n)
    out = {}
    digests = {}
    for name, a in cases.items():
        lu = np.asfortranarray(a, dtype=np.float64).copy(order="F")
        piv = np.arange(a.shape[0], dtype=np.int64)
        rlra.backend.plu_inplace(lu, piv)
        digests[name] = {"shape": list(a.shape), "lu_sha": sha_f64(lu), "piv_sha": sha(piv)}
        out[f"{name}/piv"] = piv
        if a.size <= 4096:  # small cases: full arrays; large ones: recipe + digest
            out[f"{name}/a"] = np.asfortranarray(a, dtype=np.float64)
            out[f"{name}/lu"] = lu
    np.savez_compressed(os.path.join(HERE, "gepp.npz"), **out)
    return digests


def driver_cases():
    """Small end-to-end calls of the three drivers (outputs of the reference)."""
    out = {}
    meta = {}
    a, _ = matgen.gen_decay("fast", 200, 160, seed=7)
    out["pl_a"] = a
    for v in (2, 3, 4, 5, 6):
        f = fixedrank.powerlu(a, 30, q_os=10, v=v, seed=1)
        out[f"pl_v{v}/p"], out[f"pl_v{v}/q"] = f.p, f.q
        out[f"pl_v{v}/L"], out[f"pl_v{v}/U"] = f.L, f.U
        meta[f"pl_v{v}"] = {"rel_err": core.rel_fro_error(a, fixedrank.reconstruct(f))}
    # exact rank, all parities (pkg/tests/test_fixedrank.py:50-56)
    sig = np.concatenate([np.linspace(2.0, 1.0, 8), np.zeros(35 - 8)])
    ex, _ = matgen.gen_decay("custom", 50, 35, seed=6, sigma=sig)
    out["exact_a"] = ex
    for v in (2, 3, 4, 5):
        f = fixedrank.powerlu(ex, 8, q_os=4, v=v, seed=0)
        out[f"exact_v{v}/p"], out[f"exact_v{v}/q"] = f.p, f.q
        meta[f"exact_v{v}"] = {"rel_err": core.rel_fro_error(ex, fixedrank.reconstruct(f))}
    # the v=2 basis is QR of A^T Omega (pkg/tests/test_rangefinder.py:63-68)
    b = rlra.general_power_basis_v(a, 40, 2, 9)
    out["basis_v2/V"] = b.V
    b = rlra.general_power_basis_v(a, 40, 5, 9)
    out["basis_v5/V"] = b.V
    # fixed precision (pkg/tests/test_fixedprec.py:58-78, :124-130)
    fa, _ = matgen.gen_decay("fast", 150, 150, seed=1)
    out["fp_a"] = fa
    o = fixedprec.adaptive_rank(fa, fixedprec.PrecisionParams(1e-3, 5, 60, 4), seed=0)
    out["fp/V"], out["fp/G"] = o.V, o.G
    meta["fp"] = {"rank": o.rank, "residual": o.residual_energy, "converged": o.converged}
    fac, o = fixedprec.powerlu_fp(fa, fixedprec.PrecisionParams(1e-3, 5, 60, 4), seed=0)
    out["fpfac/p"], out["fpfac/q"] = fac.p, fac.q
    meta["fpfac"] = {"rank": fac.rank,
                     "rel_err": core.rel_fro_error(fa, fixedrank.reconstruct(fac))}
    sa, _ = matgen.gen_decay("slow", 120, 120, seed=4)
    out["fp_nc_a"] = sa
    o = fixedprec.adaptive_rank(sa, fixedprec.PrecisionParams(1e-6, 10, 20, 4), seed=0)
    meta["fp_nc"] = {"rank": o.rank, "residual": o.residual_energy, "converged": o.converged}
    # single pass (pkg/tests/test_singlepass.py:72-88)
    sp_a, sigma = matgen.gen_decay("fast", 120, 100, seed=9)
    out["sp_a"] = sp_a
    f = singlepass.single_pass_lu(singlepass.DenseColumnStream(sp_a), 20, seed=0, q_os=5)
    out["sp/p"], out["sp/q"], out["sp/L"], out["sp/U"] = f.p, f.q, f.L, f.U
    meta["sp"] = {"rel_err": core.rel_fro_error(sp_a, fixedrank.reconstruct(f))}
    g, h = singlepass.stream_sketch(singlepass.DenseColumnStream(sp_a), 25, 3, panel=16)
    out["sk/G"], out["sk/H"] = g, h
    np.savez_compressed(os.path.join(HERE, "drivers.npz"), **out)
    return meta


def config_summaries():
    """Scalar summaries of the reference on C1 and C2."""
    meta = {}
    a = configs.gen_c1()
    t0 = time.perf_counter()
    f = fixedrank.powerlu(a, 50, 10, 3, 0)
    meta["C1"] = {"call": "powerlu(A, 50, 10, 3, 0)", "wall_s": time.perf_counter() - t0,
                  "rel_err": core.rel_fro_error(a, fixedrank.reconstruct(f)),
                  "p_sha": sha(f.p), "q_sha": sha(f.q)}
    np.savez_compressed(os.path.join(HERE, "c1_pq.npz"), p=f.p, q=f.q)
    if os.environ.get("GOLDEN_SKIP_C2"):
        return meta
    a = configs.gen_c2()
    pq = {}
    for v in (2, 3, 4, 5, 6):
        t0 = time.perf_counter()
        f = fixedrank.powerlu(a, 200, 20, v, 0)
        wall = time.perf_counter() - t0
        err = configs_rel_err(a, f)
        meta[f"C2_v{v}"] = {"call": f"powerlu(A, 200, 20, {v}, 0)", "wall_s": wall,
                            "rel_err": err, "p_sha": sha(f.p), "q_sha": sha(f.q)}
        pq[f"v{v}_p"], pq[f"v{v}_q"] = f.p.astype(np.int32), f.q.astype(np.int32)
        print("C2", v, wall, err, flush=True)
    np.savez_compressed(os.path.join(HERE, "c2_pq.npz"), **pq)
    return meta


def configs_rel_err(a, f):
    ap = a[f.p, :][:, f.q]
    return core.fro_norm(ap - f.L @ f.U) / core.fro_norm(a)


if __name__ == "__main__":
    meta = {"reference": f"rlra {rlra.__version__} backend={rlra.BACKEND}",
            "numpy": np.__version__}
    meta["gepp_cases"] = gepp_cases()
    meta["drivers"] = driver_cases()
    meta["configs"] = config_summaries()
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print(json.dumps(meta["configs"], indent=1))
