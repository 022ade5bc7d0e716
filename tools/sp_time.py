"""Wall and CUDA-event time of repeated device-resident single_pass_lu calls (sweep-panel size study).
usage: python tools/sp_time.py [m] [n] [reps]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2002_07138_b200 as P

m, n, reps = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (20000, 20000, 5)))
dev = torch.device("cuda", 0)
a = torch.randn(n, m, dtype=torch.float64, device=dev).t()
dm = P.DeviceMatrix(a)
for i in range(reps):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    e0.record()
    f = P.single_pass_lu(P.DeviceColumnStream(dm), 360, 0, q_os=360, panel=1024)
    e1.record()
    torch.cuda.synchronize()
    print(f"rep {i}: wall {1e3 * (time.perf_counter() - t):8.1f} ms  events {e0.elapsed_time(e1):8.1f} ms", flush=True)
