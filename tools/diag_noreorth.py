"""randlu_noreorth on the slow-decay case: where the pivots leave the
reference's (the raw chain is roundoff-dominated beyond the numerical rank)."""
import json, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import paper_2002_07138_b200 as P
from oracle import rlra_oracle as O
G = os.path.join(os.path.dirname(__file__), "..", "tests", "golden")
BL = np.load(os.path.join(G, "baselines.npz")); META = json.load(open(os.path.join(G, "baselines.json")))
for name in ["nr_slow_p2", "nr_dec_p1", "lu_slow_p2"]:
    c = META[name]; a = BL[c["a"]]
    f = getattr(P, c["fn"])(a, **c["kw"])
    dp = np.nonzero(f.p != BL[f"{name}/p"])[0]; dq = np.nonzero(f.q != BL[f"{name}/q"])[0]
    err = O.fro_norm(a - O.reconstruct(f)) / O.fro_norm(a)
    print(name, "p diff at", dp[:6], "q diff at", dq[:6], "err", err, "ref", c["rel_err"])
