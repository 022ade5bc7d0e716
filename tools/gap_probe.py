"""GPU idle time inside the C2 v=4 powerlu step (torch.profiler / CUPTI kernel
timeline): per-step span, busy time, and the largest gaps with the kernels
either side.  Usage: python tools/gap_probe.py [steps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2002_07138_b200 as P  # noqa: E402
from paper_2002_07138_b200 import configs  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
dev = torch.device("cuda", 0)
a = configs.gen_device("C2", dev)
dm = P.DeviceMatrix(a, 0)
P.set_omega_cache(True)
for _ in range(3):
    P.powerlu(dm, 200, 20, 4, 0)
torch.cuda.synchronize()
acts = [torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]
with torch.profiler.profile(activities=acts) as prof:
    for _ in range(steps):
        with torch.profiler.record_function("step"):
            P.powerlu(dm, 200, 20, 4, 0)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev = sorted(ev, key=lambda e: e.time_range.start)
ks = [(e.time_range.start, e.time_range.end, e.name) for e in ev if e.time_range.end > e.time_range.start and e.name != "step"]
span = ks[-1][1] - ks[0][0]
busy, gaps, cur = 0.0, [], ks[0][1]
busy = sum(min(e, 1e18) - s for s, e, _ in ks)
prev = ks[0]
for k in ks[1:]:
    if k[0] > prev[1]:
        gaps.append((k[0] - prev[1], prev[2][:60], k[2][:60]))
    if k[1] > prev[1]:
        prev = k
print(f"{steps} steps: span {span / 1e3:.3f} ms ({span / steps / 1e3:.3f} ms/step), kernels {len(ks)}, "
      f"busy(sum) {busy / 1e3:.3f} ms, gaps {sum(g[0] for g in gaps) / 1e3:.3f} ms in {len(gaps)}")
agg = {}
for g, a_, b_ in gaps:
    key = (a_, b_)
    n, t = agg.get(key, (0, 0.0))
    agg[key] = (n + 1, t + g)
for (a_, b_), (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{t / steps:8.1f} us/step  x{n / steps:4.1f}  {a_}  ->  {b_}")
