"""Golden vectors for the paper's comparison drivers:
randsvd, randlu, randlu_noreorth, power_basis_q, power_basis_lu_l -- outputs
of the UNMODIFIED reference (built into oracle/_ref by oracle/build_ref.sh),
on the reference tests' own inputs (pkg/tests/test_fixedrank.py) plus decay
matrices.  Writes tests/golden/baselines.npz + baselines.json.
usage: PYTHONPATH=oracle/_ref python tests/golden/make_golden_baselines.py"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle", "_ref"))
from rlra import core, fixedrank, matgen, rangefinder  # noqa: E402


def exact_rank_matrix(m, n, r, seed, best=2.0, worst=1.0):
    """pkg/tests/test_fixedrank.py:9-12."""
    sig = np.concatenate([np.linspace(best, worst, r), np.zeros(min(m, n) - r)])
    a, _ = matgen.gen_decay("custom", m, n, seed=seed, sigma=sig)
    return a


def main():
    out, meta = {}, {}
    dec, sigma = matgen.gen_decay("fast", 200, 160, seed=7)
    slow, _ = matgen.gen_decay("slow", 300, 300, seed=12)
    out["dec_a"], out["slow_a"] = dec, slow
    out["ex4_a"] = exact_rank_matrix(50, 35, 8, seed=4)
    out["ex5_a"] = exact_rank_matrix(50, 35, 8, seed=5)
    out["g_a"] = core.gaussian(0, 40, 30)
    cases = {
        "svd_dec_p1": ("randsvd", "dec_a", dict(k=30, q_os=10, p=1, seed=1)),
        "svd_dec_p2_t": ("randsvd", "dec_a", dict(k=25, q_os=5, p=2, seed=3, truncate=True)),
        "svd_g": ("randsvd", "g_a", dict(k=5, q_os=3, p=1, seed=1)),
        "svd_ex4": ("randsvd", "ex4_a", dict(k=8, q_os=4, p=1, seed=0, truncate=True)),
        "lu_dec_p0": ("randlu", "dec_a", dict(k=30, q_os=10, p=0, seed=1)),
        "lu_dec_p1": ("randlu", "dec_a", dict(k=30, q_os=10, p=1, seed=1)),
        "lu_dec_p2": ("randlu", "dec_a", dict(k=30, q_os=10, p=2, seed=2)),
        "lu_ex5": ("randlu", "ex5_a", dict(k=8, q_os=4, p=1, seed=0)),
        "lu_slow_p2": ("randlu", "slow_a", dict(k=80, q_os=10, p=2, seed=0)),
        "nr_dec_p0": ("randlu_noreorth", "dec_a", dict(k=30, q_os=10, p=0, seed=1)),
        "nr_dec_p1": ("randlu_noreorth", "dec_a", dict(k=30, q_os=10, p=1, seed=1)),
        "nr_slow_p2": ("randlu_noreorth", "slow_a", dict(k=80, q_os=10, p=2, seed=0)),
    }
    for name, (fn, an, kw) in cases.items():
        a = out[an]
        f = getattr(fixedrank, fn)(a, **kw)
        meta[name] = {"fn": fn, "a": an, "kw": kw}
        if fn == "randsvd":
            out[f"{name}/U"], out[f"{name}/S"], out[f"{name}/V"] = f.U, f.S, f.V
            meta[name]["rel_err"] = core.rel_fro_error(a, (f.U * f.S) @ f.V.T)
        else:
            out[f"{name}/p"], out[f"{name}/q"], out[f"{name}/L"], out[f"{name}/U"] = f.p, f.q, f.L, f.U
            meta[name]["rel_err"] = core.rel_fro_error(a, fixedrank.reconstruct(f))
    b = rangefinder.power_basis_q(dec, 40, 2, 9)
    out["pbq/V"] = b.V
    meta["pbq"] = {"passes": b.passes_used}
    sk = rangefinder.power_basis_lu_l(dec, 40, 1, 9)
    out["pblu/L"], out["pblu/U"], out["pblu/p"] = sk.L, sk.U, sk.p
    np.savez_compressed(os.path.join(HERE, "baselines.npz"), **out)
    with open(os.path.join(HERE, "baselines.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print(json.dumps({k: v.get("rel_err") for k, v in meta.items()}, indent=1))


if __name__ == "__main__":
    main()
