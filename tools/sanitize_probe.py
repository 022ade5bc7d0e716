"""Small invocations of every device kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): pass engine (guarded and raw, blocked),
GEPP (cooperative + blocked), CholeskyQR2 / shifted CholeskyQR3, Householder,
TRSM, RNG, SpMM, validation, the drivers.  Exits non-zero on a parity error."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2002_07138_b200 as P  # noqa: E402
from paper_2002_07138_b200 import ops, validate  # noqa: E402
from oracle import rlra_oracle as O  # noqa: E402

dev = ops.check_device()
rng = np.random.default_rng(0)
a = np.asfortranarray(rng.standard_normal((700, 500)))
ad = ops.from_numpy(a, dev)
b = ops.from_numpy(rng.standard_normal((500, 40)), dev)
bt = ops.from_numpy(rng.standard_normal((700, 40)), dev)
prep = ops.OzPrep(ad)
c = ops.to_numpy(prep.gemm(b))
assert np.abs(c - a @ ops.to_numpy(b)).max() < 1e-11
prep.gemm(bt, trans=True)
ops.OzPrep(ad, guard=False).gemm(b)
blk = ops.OzBlocked(ad, block_bytes=14 * 300 * 500, col_cap=256, cache_bytes=0, guard=False)
blk.gemm(b)
blk.gemm(bt, trans=True)
for m, n in ((600, 120), (3000, 40)):  # cooperative and blocked GEPP paths
    x = np.asfortranarray(rng.standard_normal((m, n)))
    lu, piv = x.copy(order="F"), np.arange(m, dtype=np.int64)
    P.plu_inplace(lu, piv)
    lu2, piv2 = x.copy(order="F"), np.arange(m, dtype=np.int64)
    O.plu_inplace(lu2, piv2)
    assert np.array_equal(piv, piv2) and np.array_equal(lu.view(np.int64), lu2.view(np.int64))
z = ops.from_numpy(rng.standard_normal((2000, 300)), dev)
ops.scholqr3(z)
ops.cholqr2(ops.from_numpy(rng.standard_normal((2000, 100)), dev))
qr = ops.QR(ops.from_numpy(rng.standard_normal((900, 64)), dev))
qr.q()
r = ops.as_fmat(torch.triu(torch.rand(64, 64, dtype=torch.float64, device=dev)) + 2 * torch.eye(64, dtype=torch.float64, device=dev))
ops.trsm_rt_(r, ops.from_numpy(rng.standard_normal((64, 30)), dev))
ops.trsm_un_(r, ops.from_numpy(rng.standard_normal((64, 30)), dev))
f = P.powerlu(a, 20, 10, 4, 1)
g = O.powerlu(a, 20, 10, 4, 1)
assert np.array_equal(f.p, g.p) and np.array_equal(f.q, g.q)
fp, out = P.powerlu_fp(a, P.PrecisionParams(1e-3, 5, 60, 3), 0)
sp = P.single_pass_lu(P.DenseColumnStream(a), 15, 0, q_os=5)
validate.rel_err_device(ad, P.powerlu(P.DeviceMatrix(ad), 20, 10, 3, 1))
P.randsvd(a, 10, 5, 1, 0)
import scipy.sparse as sps  # noqa: E402
P.powerlu(sps.random(400, 300, density=0.05, random_state=1, format="csr"), 10, 5, 3, 0)
torch.cuda.synchronize()
print("sanitize probe ok")
