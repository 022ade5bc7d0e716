"""Build a config's A in HBM (configs.gen_device), run the drop-in call on it,
time it with CUDA events and report rank / pivots digest / device residual.
usage: python tools/run_config.py C5 [reps]"""
import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2002_07138_b200 as P
from paper_2002_07138_b200 import configs, validate

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda", 0)
t0 = time.perf_counter()
a = configs.gen_device(name, dev)
gen_s = time.perf_counter() - t0
w = configs.WORKLOADS[name]
dm = P.DeviceMatrix(a)
P.set_omega_cache(True)


def call():
    if w.kind == "powerlu":
        return P.powerlu(dm, w.k, w.q_os, w.v, w.seed), None
    if w.kind == "powerlu_fp":
        f, out = P.powerlu_fp(dm, P.PrecisionParams(w.eps, w.b, 1024, w.v), w.seed)
        return f, out.rank
    return P.single_pass_lu(P.DeviceColumnStream(dm), w.k, w.seed, q_os=w.q_os), None


f, rank = call()
torch.cuda.synchronize()
times = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    f, rank = call()
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
if os.environ.get("BREAKDOWN"):
    from paper_2002_07138_b200 import ops

    ops.PROF.on = True
    call()
    ops.PROF.on = False
    summ = ops.PROF.summary()
    for lab, (tot, cnt) in sorted(summ.items(), key=lambda x: -x[1][0]):
        print(f"  {lab:32s} {tot:9.3f} ms  {cnt:4d} calls", file=sys.stderr)
    ops.PROF.records.clear()
err = validate.rel_err_device(a, f)
sha = lambda x: hashlib.sha256(np.ascontiguousarray(x.cpu().numpy(), dtype=np.int64).tobytes()).hexdigest()
if w.kind == "powerlu":
    passes, fact = configs.powerlu_flops(w.m, w.n, w.k, w.k + w.q_os, w.v)
    flops = passes + fact
else:
    flops = None
print(json.dumps({"config": name, "gen_s": gen_s, "ms": times, "best_ms": min(times),
                  "gflops": (flops / (min(times) / 1e3) / 1e9) if flops else None,
                  "rel_err": err, "rank": rank if rank is not None else f.rank,
                  "p_sha": sha(f.p), "q_sha": sha(f.q),
                  "mem_gb": torch.cuda.max_memory_allocated() / 1e9}))
np.savez_compressed(f"gpurun_out/{name.lower()}_gpu_pq.npz", p=f.p.cpu().numpy().astype(np.int32),
                    q=f.q.cpu().numpy().astype(np.int32))
