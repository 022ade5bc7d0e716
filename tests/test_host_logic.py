"""Host-side semantics of the drop-in API (validation, the fixed-precision
scan, restart policy, error types) against the reference's contracts and the
oracle.  CPU only: none of these launch kernels."""

import math

import numpy as np
import pytest

import paper_2002_07138_b200 as P
from oracle import rlra_oracle as O
from paper_2002_07138_b200 import configs, fixedprec


def test_params_validation():  # rlra/fixedprec.py:37-45 (pkg/tests/test_fixedprec.py:18-33)
    assert P.PrecisionParams(eps=1e-3, b=5, l=20, v=4).l == 20
    P.PrecisionParams(eps=1.0, b=1, l=1, v=2)
    for bad in (dict(eps=0.0, b=5, l=20, v=4), dict(eps=1.5, b=5, l=20, v=4),
                dict(eps=1e-3, b=0, l=20, v=4), dict(eps=1e-3, b=5, l=18, v=4),
                dict(eps=1e-3, b=5, l=0, v=4), dict(eps=1e-3, b=5, l=20, v=1)):
        with pytest.raises(ValueError):
            P.PrecisionParams(**bad)


def test_default_width():
    assert P.default_width(10, 500, 1000) == 500
    assert P.default_width(7, 100, 50) == 49
    assert P.default_width(1, 2000, 2000) == 50
    with pytest.raises(ValueError):
        P.default_width(60, 50, 50)


def unit_cols(weights):
    g = np.zeros((len(weights), len(weights)))
    for j, w in enumerate(weights):
        g[j, j] = np.sqrt(w)
    return g


def test_refine_rank_frozen():  # pkg/tests/test_fixedprec.py:41-55
    g = unit_cols([4.0, 3.0, 2.0, 1.0])
    rank, e = P.refine_rank(g, 10.0, 3.5, 0, 4)
    assert rank == 2 and e == pytest.approx(3.0, abs=1e-13)
    rank, e = P.refine_rank(g, 10.0, -1.0, 0, 4)
    assert rank == 4 and e == pytest.approx(0.0, abs=1e-13)
    g = unit_cols([5.0, 3.0, 0.0, 0.0, 2.0, 1.0, 0.0, 0.0])
    rank, e = P.refine_rank(g, 4.0, 1.5, 4, 2)
    assert rank == 6 and e == pytest.approx(1.0, abs=1e-13)


@pytest.mark.parametrize("seed", range(6))
def test_scan_matches_reference_scan(seed):
    """Our energy scan (per-column energies in, rank out) reproduces the
    reference's blocked scan (rlra/fixedprec.py:73-94) on the same G."""
    rng = np.random.default_rng(seed)
    m, l, b = 300, 60, 5
    g = rng.standard_normal((m, l)) * np.exp(-np.arange(l) / 8.0)
    total = float((rng.standard_normal((m, 80)) ** 2).sum()) + float((g ** 2).sum())
    eps = [1e-1, 1e-2, 3e-3, 1e-3, 1e-4, 0.5][seed]
    # reference formulation
    acc = eps ** 2 * total
    e = total
    ref = (l, None, False)
    for t1 in range(0, l, b):
        e_before = e
        e -= O.fro_norm(g[:, t1:t1 + b]) ** 2
        if e <= acc:
            r, e_out = O.refine_rank(g, e_before, acc, t1, b)
            ref = (r, max(e_out, 0.0), True)
            break
    else:
        ref = (l, max(e, 0.0), False)
    energies = np.array([float(g[:, j] @ g[:, j]) for j in range(l)])
    got = fixedprec.scan_energies(total, energies, eps, b, l)
    assert got[0] == ref[0] and got[2] == ref[2]
    assert abs(got[1] - ref[1]) <= 1e-12 * total


def test_restart_policy():  # rlra/fixedprec.py:166-181
    out = P.AdaptiveOutcome(20, None, None, 1.0, False)
    params = P.PrecisionParams(1e-6, 10, 20, 4)
    assert P.restart_policy(out, params, 115).l == 40
    assert P.restart_policy(out, P.PrecisionParams(1e-6, 10, 80, 4), 115).l == 110
    with pytest.raises(P.Unsatisfiable):
        P.restart_policy(out, P.PrecisionParams(1e-6, 10, 110, 4), 115)
    with pytest.raises(ValueError):
        P.restart_policy(P.AdaptiveOutcome(5, None, None, 0.0, True), params, 100)


def test_error_types_mirror_reference():  # rlra/errors.py:8-39
    e = P.RankCollapse(3, 5)
    assert (e.achieved, e.requested) == (3, 5) and "3 usable columns of 5" in str(e)
    out = P.AdaptiveOutcome(20, None, None, 4.25e-05, False)
    e = P.NotConverged(out)
    assert e.outcome is out and "full sketch width 20" in str(e)
    for cls in (P.RankCollapse, P.NotConverged, P.IllPosedPseudoinverse, P.Unsatisfiable, P.DeviceError):
        assert issubclass(cls, P.RlraError)


def test_rank_checks_raise_first_collapse():
    import torch

    from paper_2002_07138_b200.rangefinder import RankChecks

    c = RankChecks()
    c.add(torch.tensor([5]), 5)
    c.add(torch.tensor([3]), 5)
    c.add(torch.tensor([1]), 5)
    with pytest.raises(P.RankCollapse) as exc:
        c.raise_if_collapsed()
    assert exc.value.achieved == 3


def test_flop_model_matches_survey_table():
    passes, fact = configs.powerlu_flops(20000, 10000, 200, 220, 4)
    assert passes / 1e9 == pytest.approx(344.0) and fact / 1e9 == pytest.approx(7.0, abs=0.05)
    passes, fact = configs.powerlu_flops(262144, 32768, 512, 544, 4)
    assert passes / 1e9 == pytest.approx(36833.6, rel=1e-4) and fact / 1e9 == pytest.approx(357.6, rel=1e-3)


def test_gaussian_is_reference_stream():  # rlra/core.py:33-48, prefix property
    a = P.gaussian(5, 7, 3)
    assert np.array_equal(a, O.gaussian(5, 7, 3))
    assert np.array_equal(P.gaussian(5, 7, 5)[:, :3], a)
