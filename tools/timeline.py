"""Timeline of one warm call of a config (device-built A): every C-ABI call's
start offset and duration (CUDA events on the launching stream) plus per-label
totals.  usage: python tools/timeline.py C3 [min_us]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2002_07138_b200 as P  # noqa: E402
from paper_2002_07138_b200 import configs, ops  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
min_us = float(sys.argv[2]) if len(sys.argv) > 2 else 50.0
w = configs.WORKLOADS[name]
dev = torch.device("cuda", 0)
dm = P.DeviceMatrix(configs.gen_device(name, dev))
P.set_omega_cache(True)
if w.kind == "powerlu":
    call = lambda: P.powerlu(dm, w.k, w.q_os, w.v, w.seed)  # noqa: E731
elif w.kind == "powerlu_fp":
    call = lambda: P.powerlu_fp(dm, P.PrecisionParams(w.eps, w.b, 1024, w.v), w.seed)  # noqa: E731
else:
    call = lambda: P.single_pass_lu(P.DeviceColumnStream(dm), w.k, w.seed, q_os=w.q_os)  # noqa: E731
call()
call()
torch.cuda.synchronize()
ops.PROF.records.clear()
ops.PROF.on = True
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
call()
e1.record(st)
torch.cuda.synchronize()
ops.PROF.on = False
print(f"{name}: total {e0.elapsed_time(e1):.3f} ms")
tot = {}
for lab, a0, a1 in ops.PROF.records:
    d = a0.elapsed_time(a1)
    t, c = tot.get(lab, (0.0, 0))
    tot[lab] = (t + d, c + 1)
    if d * 1e3 >= min_us:
        print(f"  +{e0.elapsed_time(a0):9.3f} ms  {d:8.3f} ms  {lab}")
print("per label:")
for lab, (t, c) in sorted(tot.items(), key=lambda kv: -kv[1][0]):
    print(f"  {lab:34s} {t:8.3f} ms  {c:4d} calls")
