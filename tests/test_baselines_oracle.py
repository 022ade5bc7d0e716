"""Pin the oracle's restatement of the paper's comparison drivers (randsvd,
randlu, randlu_noreorth, power_basis_q, power_basis_lu_l; SURVEY.md §8(f)
row 1) against the golden outputs of the unmodified reference
(tests/golden/make_golden_baselines.py).  CPU only."""

import json
import os

import numpy as np
import pytest

from oracle import rlra_oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
META = json.load(open(os.path.join(GOLD, "baselines.json")))
BL = np.load(os.path.join(GOLD, "baselines.npz"))
CASES = sorted(k for k in META if "fn" in META[k])


@pytest.mark.parametrize("name", CASES)
def test_oracle_baseline_matches_reference(name):
    c = META[name]
    f = getattr(O, c["fn"])(BL[c["a"]], **c["kw"])
    if c["fn"] == "randsvd":
        for fld in "USV":
            assert np.array_equal(getattr(f, fld), BL[f"{name}/{fld}"])
    else:
        for fld in ("p", "q", "L", "U"):
            assert np.array_equal(getattr(f, fld), BL[f"{name}/{fld}"])


def test_oracle_power_bases_match_reference():
    a = BL["dec_a"]
    b = O.power_basis_q(a, 40, 2, 9)
    assert b.passes_used == META["pbq"]["passes"] == 5
    assert np.array_equal(b.V, BL["pbq/V"])
    sk = O.power_basis_lu_l(a, 40, 1, 9)
    assert np.array_equal(sk.L, BL["pblu/L"]) and np.array_equal(sk.U, BL["pblu/U"])
    assert np.array_equal(sk.p, BL["pblu/p"])


def test_oracle_noreorth_equals_randlu_at_p0():
    """pkg/tests/test_fixedrank.py:101-108."""
    a = O.gaussian(11, 40, 30)
    f1 = O.randlu(a, 6, q_os=4, p=0, seed=3)
    f2 = O.randlu_noreorth(a, 6, q_os=4, p=0, seed=3)
    for fld in ("L", "U", "p", "q"):
        assert np.array_equal(getattr(f1, fld), getattr(f2, fld))
