"""Consecutive e2e powerlu calls (pinned host A -> NumPy factors): per-call
CUDA-event time and host wall time, to expose per-call overheads."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2002_07138_b200 as P
from paper_2002_07138_b200 import configs
a = configs.gen_c2()
m, n = a.shape
pinned = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
ah = pinned.numpy().T
ah[...] = a
P.set_omega_cache(False)
fh = P.powerlu(ah, 200, 20, 4, 0)
torch.cuda.synchronize()
st = torch.cuda.current_stream()
for i in range(6):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record(st)
    fh = P.powerlu(ah, 200, 20, 4, 0)
    e1.record(st); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"call {i}: events {e0.elapsed_time(e1):6.2f} ms  host {1e3 * (t1 - t0):6.2f} ms", flush=True)
P.set_omega_cache(True)
for i in range(3):
    t0 = time.perf_counter(); fh = P.powerlu(ah, 200, 20, 4, 0); torch.cuda.synchronize()
    print(f"cached-omega call {i}: host {1e3 * (time.perf_counter() - t0):6.2f} ms", flush=True)
