"""Time the device GEPP (librlra_b200, no tracing) on sketch shapes with CUDA
events.  usage: python tools/time_getrf.py [m,n ...]   (RLRA_B200_LU_FULL=1
selects the cooperative one-launch GEPP for eligible shapes)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_07138_b200 import ops  # noqa: E402

shapes = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]] or [(20000, 220), (10000, 220), (20000, 200),
                                                                          (10000, 200)]
dev = ops.check_device()
for m, n in shapes:
    a0 = torch.randn((n, m), dtype=torch.float64, device=dev).t()  # column-major m x n
    times = []
    for rep in range(6):
        a = ops.as_fmat(a0.clone())  # clone keeps the column-major strides
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ops.getrf_(a)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) * 1e3)
    print(f"getrf {m} x {n}: best {min(times[1:]):8.1f} us  median {sorted(times[1:])[2]:8.1f} us")
