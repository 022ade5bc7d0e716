"""Debug helper: device GEPP vs the oracle on one random shape; prints the
first differences.  usage: python tools/diag_full.py m n seed"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import rlra_oracle as O  # noqa: E402
from paper_2002_07138_b200 import ops  # noqa: E402

m, n, seed = (int(v) for v in sys.argv[1:4])
a = np.random.default_rng(seed).standard_normal((m, n))
if len(sys.argv) > 4 and n > 40:  # the parity test's exact zero pivots (tests/test_gepp_gpu.py)
    a[:, 33] = a[:, 5]
    a[:, 40] = 0.0
lu_ref = np.asfortranarray(a).copy(order="F")
piv_ref = np.arange(m, dtype=np.int64)
O.plu_inplace(lu_ref, piv_ref)
d = ops.from_numpy(a, ops.check_device())
piv, cnt = ops.getrf_(d)
lu = ops.to_numpy(d)
piv = piv.cpu().numpy()
print(m, n, "piv equal", np.array_equal(piv, piv_ref), "lu bit-equal",
      np.array_equal(lu.view(np.int64), lu_ref.view(np.int64)))
bad = np.argwhere(lu.view(np.int64) != lu_ref.view(np.int64))
if len(bad):
    cols = np.unique(bad[:, 1])
    print("bad cols", cols[:12], "n bad", len(bad))
    r, c = bad[0]
    print("first bad", r, c, lu[r, c], lu_ref[r, c])
    print("bad rows", np.unique(bad[:, 0])[:20])
print("piv diff at", np.nonzero(piv != piv_ref)[0][:10])
