"""Golden outputs of the reference on inputs that stress the pass products'
numerics: integer-valued exact-rank matrices (exact cancellation can make a
pivot exactly 0.0), sketches wider than the rank (pass-through vs
RankCollapse, pkg/src/rlra/rangefinder.py:55-64), graded rows / columns and
extreme magnitudes (the int8 engine's dynamic-range guard).

Run in the build container after oracle/build_ref.sh:

    python tests/golden/make_golden_guard.py

Writes tests/golden/guard_cases.npz (inputs + p, q, L, U or the exception
raised) and guard_cases.json (rel_err, outcome).  The unmodified reference
(oracle/_ref, compiled backend) produces every number.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(REPO, "oracle", "_ref"))
os.environ["RLRA_BACKEND"] = "compiled"

import rlra  # noqa: E402  (the reference, unmodified)
from rlra import core, errors, fixedrank  # noqa: E402

assert rlra.BACKEND == "compiled"


def cases():
    out = {}
    # pkg/tests/test_cli.py:76-89: integer exact-rank-5, powerlu k=5, q_os=0, v=3
    rng = np.random.default_rng(0)
    picker = np.zeros((60, 5))
    picker[np.arange(60), rng.integers(0, 5, 60)] = 1.0
    a = picker @ rng.integers(1, 9, size=(5, 40)).astype(np.float64)
    out["int_rank5"] = (a, 5, 0, 3, 0)
    # the same matrix with a sketch wider than the rank: l = 12 > 5
    for v in (2, 3, 4):
        out[f"int_rank5_l12_v{v}"] = (a, 8, 4, v, 1)
    # a larger integer low-rank matrix (small integer factors, exact products)
    rng = np.random.default_rng(11)
    a2 = rng.integers(-3, 4, size=(300, 7)).astype(np.float64) @ rng.integers(-3, 4, size=(7, 200)).astype(np.float64)
    for v in (2, 3, 4, 5):
        out[f"int_rank7_v{v}"] = (a2, 7, 3, v, 2)
    # graded rows and columns (10 decades each): the guard sends these
    # products to the DMMA GEMM
    rng = np.random.default_rng(12)
    u, _ = np.linalg.qr(rng.standard_normal((400, 40)))
    w, _ = np.linalg.qr(rng.standard_normal((300, 40)))
    base = (u * np.exp(-np.arange(40) / 4.0)) @ w.T
    dr = 10.0 ** rng.uniform(-10, 0, size=(400, 1))
    dc = 10.0 ** rng.uniform(-10, 0, size=(1, 300))
    out["graded_rows"] = (np.asfortranarray(base * dr), 15, 5, 3, 3)
    out["graded_cols"] = (np.asfortranarray(base * dc), 15, 5, 4, 3)
    # extreme magnitudes (norms far outside the engine's range)
    out["tiny"] = (np.asfortranarray(base * 1e-140), 15, 5, 3, 4)
    out["huge"] = (np.asfortranarray(base * 1e150), 15, 5, 3, 4)
    return out


def order_outcomes(a, k, q_os, v, seed):
    """Outcome of the reference's algorithm (the oracle restatement) when its
    products sum over K in other legitimate orders: reversed, K-chunks of 64,
    reversed chunks of 32.  A case whose pass-through / RankCollapse outcome
    changes with the order is rounding-dependent, not a parity target."""
    sys.path.insert(0, REPO)
    from oracle import rlra_oracle as O

    def rev(x, y):
        return np.ascontiguousarray(x[:, ::-1]) @ np.ascontiguousarray(y[::-1])

    def chunk(x, y, c=64, reverse=False):
        out = np.zeros((x.shape[0], y.shape[1]))
        starts = range(0, x.shape[1], c)
        for k0 in (reversed(starts) if reverse else starts):
            out += x[:, k0:k0 + c] @ y[k0:k0 + c]
        return out

    res = []
    for mm in (np.matmul, rev, chunk, lambda x, y: chunk(x, y, 32, True)):
        l = k + q_os
        m, n = a.shape
        try:
            if v % 2 == 0:
                x = mm(a.T, O.gaussian(seed, m, l))
                if v == 2:
                    O._qr_basis(x)
                    res.append("ok")
                    continue
                w = O._lu_basis(x)
            else:
                w = O.gaussian(seed, n, l)
            half = (v - 1) // 2
            for i in range(1, half + 1):
                w = O._lu_basis(mm(a, w))
                if i == half:
                    O._qr_basis(mm(a.T, w))
                else:
                    w = O._lu_basis(mm(a.T, w))
            res.append("ok")
        except O.OracleRankCollapse as e:
            res.append(f"RankCollapse:{e.achieved}")
    return res


def main():
    arrays, meta = {}, {}
    for name, (a, k, q_os, v, seed) in cases().items():
        arrays[f"{name}/a"] = a
        rec = {"k": k, "q_os": q_os, "v": v, "seed": seed, "order_outcomes": order_outcomes(a, k, q_os, v, seed)}
        try:
            f = fixedrank.powerlu(a, k, q_os, v, seed)
        except errors.RankCollapse as e:
            rec.update(outcome="RankCollapse", achieved=int(e.achieved), requested=int(e.requested))
        else:
            rec.update(outcome="ok", rel_err=float(core.rel_fro_error(a, fixedrank.reconstruct(f))))
            arrays[f"{name}/p"] = f.p
            arrays[f"{name}/q"] = f.q
            arrays[f"{name}/L"] = f.L
            arrays[f"{name}/U"] = f.U
        meta[name] = rec
        print(name, rec)
    np.savez_compressed(os.path.join(HERE, "guard_cases.npz"), **arrays)
    with open(os.path.join(HERE, "guard_cases.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
