"""conftest for running the REFERENCE's own hot-path test files against
paper_2002_07138_b200 (SURVEY.md §4 "How the build should test", item 1).

tests/test_reference_suite_gpu.py copies the reference's test files (built
into oracle/_ref/tests by oracle/build_ref.sh) into a scratch directory next to
this file (renamed conftest.py) and runs pytest there.  The real reference
package is imported (oracle/_ref) and its hot-path entry points are replaced
by adapters onto the B200 package:

  fixedrank   powerlu, lu_from_projection, randsvd, randlu, randlu_noreorth,
              range_agreement
  fixedprec   adaptive_rank, powerlu_fp, refine_rank, default_width, restart_policy
  rangefinder general_power_basis_v, power_basis_v, power_basis_q, power_basis_lu_l
  singlepass  stream_sketch, single_pass_lu

Adapters pass the test's arguments through unchanged (NumPy arrays, the
reference's accessors and column streams, its PrecisionParams / PowerParams),
return the reference's result classes with NumPy fields, and re-raise the
B200 package's exceptions as the reference's classes with the same
attributes.  Everything else (core, matgen, accessors, kernels, errors, cli,
the reference's validation helpers) stays the reference's own code.
"""

import functools
import os
import sys

REPO = os.environ["RLRA_B200_REPO"]
sys.path.insert(0, os.path.join(REPO, "oracle", "_ref"))
sys.path.insert(0, REPO)
os.environ.setdefault("RLRA_BACKEND", "compiled")

import numpy as np  # noqa: E402
import torch  # noqa: E402

import rlra  # noqa: E402  (the unmodified reference)
from rlra import errors as R_err  # noqa: E402
from rlra import fixedprec as R_fp  # noqa: E402
from rlra import fixedrank as R_fr  # noqa: E402
from rlra import rangefinder as R_rf  # noqa: E402
from rlra import singlepass as R_sp  # noqa: E402

import paper_2002_07138_b200 as P  # noqa: E402
from paper_2002_07138_b200 import errors as P_err  # noqa: E402

ALIASED = []
CALLS = {}


def _np(x):
    if isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy()
    return x


def _convert(out):
    name = type(out).__name__
    if name == "LowRankLU":
        return R_fr.LowRankLU(_np(out.p), _np(out.q), _np(out.L), _np(out.U), out.rank)
    if name == "LowRankSVD":
        return R_fr.LowRankSVD(_np(out.U), _np(out.S), _np(out.V))
    if name == "AdaptiveOutcome":
        return R_fp.AdaptiveOutcome(out.rank, _np(out.V), _np(out.G), out.residual_energy, out.converged)
    if name == "RangeBasis":
        return R_rf.RangeBasis(_np(out.V), out.passes_used)
    if name == "SketchLU":
        return R_rf.SketchLU(_np(out.L), _np(out.U), _np(out.p))
    if name == "SketchPair":
        return R_sp.SketchPair(_np(out.G), _np(out.H))
    if isinstance(out, tuple):
        return type(out)(_convert(x) for x in out) if type(out) is tuple else out
    return _np(out)


def _adapter(fn, qual):
    @functools.wraps(fn)
    def call(*args, **kw):
        CALLS[qual] = CALLS.get(qual, 0) + 1
        try:
            return _convert(fn(*args, **kw))
        except P_err.RankCollapse as e:
            raise R_err.RankCollapse(e.achieved, e.requested) from None
        except P_err.NotConverged as e:
            raise R_err.NotConverged(_convert(e.outcome)) from None
        except P_err.IllPosedPseudoinverse as e:
            raise R_err.IllPosedPseudoinverse(str(e)) from None
        except P_err.Unsatisfiable as e:
            raise R_err.Unsatisfiable(str(e)) from None

    call.__b200__ = True
    return call


for mod, names in ((R_fr, ["powerlu", "lu_from_projection", "randsvd", "randlu", "randlu_noreorth",
                           "range_agreement"]),
                   (R_fp, ["adaptive_rank", "powerlu_fp", "refine_rank", "default_width", "restart_policy"]),
                   (R_rf, ["general_power_basis_v", "power_basis_v", "power_basis_q", "power_basis_lu_l"]),
                   (R_sp, ["stream_sketch", "single_pass_lu"])):
    for nm in names:
        qual = f"{mod.__name__}.{nm}"
        setattr(mod, nm, _adapter(getattr(P, nm), qual))
        ALIASED.append(qual)


def pytest_terminal_summary(terminalreporter):
    import json

    terminalreporter.write_line(f"rlra hot path aliased to paper_2002_07138_b200 ({len(ALIASED)} entry points)")
    terminalreporter.write_line("b200 calls " + json.dumps(CALLS, sort_keys=True))
