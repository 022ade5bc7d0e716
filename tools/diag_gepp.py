import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import rlra_oracle as O
from paper_2002_07138_b200 import ops

for (m, n, seed) in [(65, 64, 4), (300, 120, 0), (40, 40, 1), (100, 64, 2), (64, 33, 3)]:
    a = np.random.default_rng(seed).standard_normal((m, n))
    lu_ref = np.asfortranarray(a).copy(order="F"); piv_ref = np.arange(m, dtype=np.int64)
    O.plu_inplace(lu_ref, piv_ref)
    d = ops.from_numpy(a, ops.check_device())
    piv, _ = ops.getrf_(d)
    lu = ops.to_numpy(d); piv = piv.cpu().numpy()
    bad = np.argwhere(lu != lu_ref)
    pd = np.nonzero(piv != piv_ref)[0]
    print(m, n, "piv diff at", pd[:10], "n elems diff", len(bad))
    if len(bad):
        cols = sorted(set(bad[:, 1].tolist()))
        print("  first bad cols", cols[:10], "rows of first col", bad[bad[:, 1] == cols[0]][:10, 0].tolist())
        c = cols[0]; r = bad[bad[:, 1] == c][0, 0]
        print("  val", lu[r, c], lu_ref[r, c])
