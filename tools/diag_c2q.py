"""C2 column-pivot diagnosis: GPU determinism across repeats, comparison with
the golden q (reference run in the build container) and with the reference
run on this host; prints the pivot margin at the first differing step."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle", "_ref"))
import paper_2002_07138_b200 as P
from paper_2002_07138_b200 import configs

v = int(sys.argv[1]) if len(sys.argv) > 1 else 4
a = configs.gen_c2()
pq = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "c2_pq.npz"))
gq = pq[f"v{v}_q"]
dm = P.DeviceMatrix(a)
qs = []
for r in range(4):
    f = P.powerlu(dm, 200, 20, v, 0).to_numpy()
    qs.append(f.q)
    d = np.nonzero(f.q != gq)[0]
    print(f"run {r}: p==golden {np.array_equal(f.p, pq[f'v{v}_p'])} q==golden {d.size == 0} first diff {d[:3]}", flush=True)
print("gpu deterministic:", all(np.array_equal(qs[0], x) for x in qs))
import rlra
fr = rlra.powerlu(a, 200, 20, v, 0)
print("host ref q == golden:", np.array_equal(fr.q, gq), " host ref q == gpu:", np.array_equal(fr.q, qs[0]))
# margin: recompute the Bt GEPP on the host from the reference's basis to see the tie
basis = rlra.general_power_basis_v(a, 220, v, 0)
vk = basis.V[:, :200]
g = a @ vk
l1, u1, p1 = rlra.plu(g)
bt = (u1 @ vk.T).T
lu = bt.copy(order="F"); piv = np.arange(bt.shape[0], dtype=np.int64)
# manual GEPP tracking the top-2 margin per step
x = bt.copy()
m, k = x.shape
perm = np.arange(m)
worst = (1e9, -1)
for j in range(k):
    col = np.abs(x[j:, j])
    o = np.argsort(-col)[:2]
    if col[o[0]] > 0:
        rel = (col[o[0]] - col[o[1]]) / col[o[0]]
        if rel < worst[0]:
            worst = (rel, j)
    i = j + o[0]
    x[[j, i]] = x[[i, j]]
    perm[[j, i]] = perm[[i, j]]
    if x[j, j] != 0:
        x[j + 1:, j] /= x[j, j]
        x[j + 1:, j + 1:] -= np.outer(x[j + 1:, j], x[j, j + 1:])
print("smallest relative top-2 pivot margin in GEPP(Bt): %.3e at step %d" % worst)
