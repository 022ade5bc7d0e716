"""The bench's e2e loop (pinned host A in, NumPy factors out, Omega redrawn)
with per-step CUDA-event times, to see its spread.  usage: python tools/e2e_loop.py [steps]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2002_07138_b200 as P  # noqa: E402
from paper_2002_07138_b200 import configs  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
a = configs.gen_c2()
m, n = a.shape
pinned = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
ah = pinned.numpy().T
ah[...] = a
P.set_omega_cache(False)
for _ in range(3):
    P.powerlu(ah, 200, 20, 4, 0)
torch.cuda.synchronize()
st = torch.cuda.current_stream()
ts = []
for _ in range(steps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(st)
    P.powerlu(ah, 200, 20, 4, 0)
    e1.record(st)
    torch.cuda.synchronize()
    ts.append((e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3))
for d, w in ts:
    print(f"e2e step {d:8.3f} ms (host wall {w:8.3f})")
print("mean", sum(d for d, _ in ts) / len(ts))
