"""Bit-exactness + timing of the device GEPP at wide sketch shapes (n up to
1024, the one-launch cluster kernel's range) against the oracle."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import rlra_oracle as O
from paper_2002_07138_b200 import ops
dev = ops.check_device()
for (m, n, seed) in [(16384, 1024, 0), (4000, 700, 1), (24576, 512, 2), (8192, 300, 3)]:
    a = np.random.default_rng(seed).standard_normal((m, n))
    if n > 40:
        a[:, 33] = a[:, 5]; a[:, 40] = 0.0
    lu_ref = np.asfortranarray(a).copy(order="F"); piv_ref = np.arange(m, dtype=np.int64)
    t0 = time.perf_counter(); O.plu_inplace(lu_ref, piv_ref); tc = time.perf_counter() - t0
    bad = 0; ts = []
    for r in range(4):
        d = ops.from_numpy(a, dev); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); piv, cnt = ops.getrf_(d); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
        ok = np.array_equal(piv.cpu().numpy(), piv_ref) and np.array_equal(ops.to_numpy(d).view(np.int64), lu_ref.view(np.int64))
        bad += not ok
    print(f"{m}x{n}: {bad}/4 mismatches, best {min(ts[1:]):.2f} ms (oracle {tc:.1f} s)", flush=True)
