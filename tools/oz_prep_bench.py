"""Time ops.OzPrep (norms + residues of A) at the C2 shape with CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2002_07138_b200 import ops
m, n = (int(x) for x in sys.argv[1:3]) if len(sys.argv) > 2 else (20000, 10000)
a = torch.randn(n, m, dtype=torch.float64, device="cuda").t()
ops.OzPrep(a)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    p = ops.OzPrep(a)
    del p
e1.record()
torch.cuda.synchronize()
print(f"OzPrep {m}x{n}: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us")
