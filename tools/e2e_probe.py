"""Timeline of one e2e powerlu call (pinned host A -> NumPy factors): every
C-ABI call's start offset and duration relative to the call's start (CUDA
events on the launching stream), plus the host wall time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2002_07138_b200 as P
from paper_2002_07138_b200 import configs, ops

a = configs.gen_c2()
m, n = a.shape
pinned = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
ah = pinned.numpy().T
ah[...] = a
P.set_omega_cache(False)
for _ in range(2):
    P.powerlu(ah, 200, 20, 4, 0)
torch.cuda.synchronize()
ops.PROF.on = True
st = torch.cuda.current_stream()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record(st)
f = P.powerlu(ah, 200, 20, 4, 0)
e1.record(st)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) * 1e3
ops.PROF.on = False
print(f"total {e0.elapsed_time(e1):.2f} ms (host wall {wall:.2f} ms)")
for lab, a0, a1 in ops.PROF.records:
    print(f"  +{e0.elapsed_time(a0):8.3f} ms  {a0.elapsed_time(a1):7.3f} ms  {lab}")
