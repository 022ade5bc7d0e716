"""Repeatability of the device GEPP against the oracle (A/B library builds via
RLRA_B200_LIB): each shape factored several times; prints mismatches."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from oracle import rlra_oracle as O
from paper_2002_07138_b200 import ops

dev = ops.check_device()
reps = int(os.environ.get("REPS", "5"))
bad = 0
for (m, n, seed) in [(700, 64, 0), (2000, 60, 12), (10000, 220, 1), (20000, 220, 0), (16384, 256, 3), (24576, 256, 10)]:
    a = np.random.default_rng(seed).standard_normal((m, n))
    lu_ref = np.asfortranarray(a).copy(order="F"); piv_ref = np.arange(m, dtype=np.int64)
    O.plu_inplace(lu_ref, piv_ref)
    fails = 0
    for r in range(reps):
        d = ops.from_numpy(a, dev)
        piv, cnt = ops.getrf_(d)
        lu = ops.to_numpy(d); p = piv.cpu().numpy()
        ok = np.array_equal(p, piv_ref) and np.array_equal(lu.view(np.int64), lu_ref.view(np.int64))
        fails += not ok
    bad += fails
    print(f"{os.environ.get('TAG','')} {m}x{n}: {fails}/{reps} mismatches", flush=True)
print(f"{os.environ.get('TAG','')} TOTAL mismatches {bad}")
