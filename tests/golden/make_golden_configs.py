"""Golden summaries of the REFERENCE on the large configs C3 and C4 (and C5
when run on a host with > 150 GB RAM).

    python tests/golden/make_golden_configs.py C3 C4        # build container
    python tests/golden/make_golden_configs.py C5           # GPU box host (196 GB)

Imports the unmodified reference (oracle/_ref, compiled backend), builds A with
the SURVEY.md Appendix A recipe (paper_2002_07138_b200/configs.py, host NumPy),
runs the reference call, and writes <config>_pq.npz (p, q as int32) plus a
JSON summary (rank, rel_err via a blocked residual, wall time) into
tests/golden/.
"""

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

from oracle.rlra_oracle import rel_fro_error_factor  # noqa: E402
from paper_2002_07138_b200 import configs  # noqa: E402

assert rlra.BACKEND == "compiled"


def run(name):
    t0 = time.perf_counter()
    if name == "C3":
        a = configs.gen_c3()
    elif name == "C4":
        a = configs.gen_c4()
    elif name == "C5":
        a = configs.gen_c5()
    else:
        raise SystemExit(name)
    gen_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    meta = {"gen_s": gen_s}
    if name == "C3":
        fac, out = rlra.powerlu_fp(a, rlra.PrecisionParams(1e-6, 64, 1024, 3), 0)
        meta.update(call="powerlu_fp(A, PrecisionParams(1e-6, 64, 1024, 3), 0)", rank=out.rank,
                    residual=out.residual_energy)
    elif name == "C4":
        fac = rlra.single_pass_lu(rlra.DenseColumnStream(a), 360, 0, q_os=360)
        meta.update(call="single_pass_lu(DenseColumnStream(A), 360, 0, q_os=360)")
    else:
        fac = rlra.powerlu(a, 512, 32, 4, 0)
        meta.update(call="powerlu(A, 512, 32, 4, 0)")
    meta["wall_s"] = time.perf_counter() - t0
    meta["rel_err"] = rel_fro_error_factor(a, fac)
    meta["rank"] = int(fac.rank)
    out_dir = os.environ.get("GOLDEN_OUT", HERE)
    np.savez_compressed(os.path.join(out_dir, f"{name.lower()}_pq.npz"), p=fac.p.astype(np.int32),
                        q=fac.q.astype(np.int32))
    path = os.path.join(out_dir, "golden_configs.json")
    allm = json.load(open(path)) if os.path.exists(path) else {}
    allm[name] = meta
    with open(path, "w") as fh:
        json.dump(allm, fh, indent=1, sort_keys=True)
    print(name, json.dumps(meta), flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:]:
        run(nm)
