"""Pin the oracle (oracle/gepp.c + oracle/rlra_oracle.py) against the golden
vectors produced by the reference itself (tests/golden/make_golden.py), and --
when the unmodified reference is built in oracle/_ref -- against the live
reference.  CPU only."""

import hashlib
import json
import os
import sys

import numpy as np
import pytest

from oracle import rlra_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")
META = json.load(open(os.path.join(GOLD, "golden.json")))
GEPP = np.load(os.path.join(GOLD, "gepp.npz"))
DRV = np.load(os.path.join(GOLD, "drivers.npz"))

sys.path.insert(0, GOLD)
from make_golden_inputs import gepp_input  # noqa: E402


def sha_f64(a):
    return hashlib.sha256(np.asfortranarray(a, dtype=np.float64).tobytes(order="F")).hexdigest()


def sha_i64(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


@pytest.mark.parametrize("name", sorted(META["gepp_cases"]))
def test_oracle_gepp_bit_exact_vs_reference(name):
    a = gepp_input(name, GEPP)
    lu = np.asfortranarray(a, dtype=np.float64).copy(order="F")
    piv = np.arange(a.shape[0], dtype=np.int64)
    O.plu_inplace(lu, piv)
    d = META["gepp_cases"][name]
    assert list(a.shape) == d["shape"]
    assert sha_f64(lu) == d["lu_sha"]
    assert sha_i64(piv) == d["piv_sha"]
    assert np.array_equal(piv, GEPP[f"{name}/piv"])


def test_oracle_frozen_2x2_and_tie():
    f = O.plu(np.array([[0.0, 1.0], [2.0, 3.0]]))
    assert np.array_equal(f.p, [1, 0])
    assert np.array_equal(f.U, np.array([[2.0, 3.0], [0.0, 1.0]]))
    f = O.plu(np.array([[1.0, 5.0], [2.0, 6.0], [-2.0, 7.0]]))
    assert f.p[0] == 1  # first maximum wins (pkg/tests/test_backend.py:53-59)


@pytest.mark.parametrize("v", [2, 3, 4, 5, 6])
def test_oracle_powerlu_vs_reference(v):
    a = DRV["pl_a"]
    f = O.powerlu(a, 30, q_os=10, v=v, seed=1)
    assert np.array_equal(f.p, DRV[f"pl_v{v}/p"])
    assert np.array_equal(f.q, DRV[f"pl_v{v}/q"])
    np.testing.assert_allclose(f.L, DRV[f"pl_v{v}/L"], rtol=0, atol=1e-12 * np.abs(f.L).max())
    np.testing.assert_allclose(f.U, DRV[f"pl_v{v}/U"], rtol=0, atol=1e-12 * np.abs(f.U).max())
    err = O.rel_fro_error_factor(a, f)
    assert abs(err - META["drivers"][f"pl_v{v}"]["rel_err"]) <= 1e-14


def test_oracle_adaptive_rank_vs_reference():
    o = O.adaptive_rank(DRV["fp_a"], 1e-3, 5, 60, 4, seed=0)
    ref = META["drivers"]["fp"]
    assert o.rank == ref["rank"] and o.converged
    assert abs(o.residual_energy - ref["residual"]) <= 1e-12
    o = O.adaptive_rank(DRV["fp_nc_a"], 1e-6, 10, 20, 4, seed=0)
    assert o.rank == 20 and not o.converged


def test_oracle_single_pass_vs_reference():
    f = O.single_pass_lu(DRV["sp_a"], 20, seed=0, q_os=5)
    assert np.array_equal(f.p, DRV["sp/p"]) and np.array_equal(f.q, DRV["sp/q"])
    assert abs(O.rel_fro_error_factor(DRV["sp_a"], f) - META["drivers"]["sp"]["rel_err"]) <= 1e-12
    g, h = O.stream_sketch(DRV["sp_a"], 25, 3, panel=16)
    np.testing.assert_allclose(g, DRV["sk/G"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(h, DRV["sk/H"], rtol=0, atol=1e-12)


def test_oracle_c1_summary_vs_reference():
    from paper_2002_07138_b200 import configs

    a = configs.gen_c1()
    f = O.powerlu(a, 50, 10, 3, 0)
    ref = META["configs"]["C1"]
    assert sha_i64(f.p) == ref["p_sha"] and sha_i64(f.q) == ref["q_sha"]
    assert abs(O.rel_fro_error_factor(a, f) - ref["rel_err"]) <= 1e-12


REF = os.path.join(os.path.dirname(HERE), "oracle", "_ref")


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "rlra")), reason="oracle/_ref not built")
def test_oracle_matches_live_reference_gepp():
    sys.path.insert(0, REF)
    os.environ.setdefault("RLRA_BACKEND", "compiled")
    import rlra

    rng = np.random.default_rng(11)
    for (m, n) in [(97, 31), (31, 97), (400, 64)]:
        a = rng.standard_normal((m, n))
        a[:, 3] = a[:, 1]  # exact dependent column -> zero pivot
        f1 = rlra.kernels.plu(a)
        f2 = O.plu(a)
        assert np.array_equal(f1.L, f2.L) and np.array_equal(f1.U, f2.U)
        assert np.array_equal(f1.p, f2.p)
