"""Per-piece timing of CholeskyQR2 at the C2 sketch shape (10000 x 220)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_07138_b200 import ops  # noqa: E402

dev = torch.device("cuda", 0)
n, l = (int(x) for x in sys.argv[1:3]) if len(sys.argv) > 2 else (10000, 220)
x = ops.from_numpy(np.random.default_rng(0).standard_normal((n, l)) * np.logspace(0, -4, l), dev)
flag = torch.zeros(1, dtype=torch.int32, device=dev)
rinv = ops.fmat(l, l, dev)


def t(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


g = ops.matmul(x, x, ta=True)
print("gram TN   %.1f us" % t(lambda: ops.matmul(x, x, ta=True)))
gs = [g.clone() for _ in range(25)]
it = iter(gs)
print("chol_inv  %.1f us (incl. nothing else)" % t(lambda: ops.chol_inv(next(it), rinv, flag, 1e8)))
print("flag", int(flag.item()))
print("Z Rinv NN %.1f us" % t(lambda: ops.matmul(x, rinv)))
print("cholqr2   %.1f us" % t(lambda: ops.cholqr2(x)))
qr_t = t(lambda: ops.QR(x.clone()).q(), reps=5)
print("householder geqrf+orgqr %.1f us" % qr_t)
