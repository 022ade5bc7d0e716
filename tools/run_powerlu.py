"""One warm powerlu of a config for profiling launch lists (ncu).  Usage:
python tools/run_powerlu.py [C2] [v] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2002_07138_b200 as P
from paper_2002_07138_b200 import configs

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
w = configs.WORKLOADS[cfg]
v = int(sys.argv[2]) if len(sys.argv) > 2 else w.v
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
if cfg == "C2":
    m, n = w.m, w.n
    rng = torch.Generator().manual_seed(0)
    a = torch.randn((n, m), generator=rng, dtype=torch.float64).numpy().T  # fast stand-in, same shape
else:
    a = {"C1": configs.gen_c1}[cfg]()
dm = P.DeviceMatrix(a)
P.set_omega_cache(True)
P.powerlu(dm, w.k, w.q_os, v, w.seed)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("timed")
for _ in range(reps):
    P.powerlu(dm, w.k, w.q_os, v, w.seed)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("ok")
