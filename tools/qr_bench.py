"""Householder QR (geqrf + orgqr, K4) timing at a sketch shape."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2002_07138_b200 import ops
n, l = (int(x) for x in sys.argv[1:3]) if len(sys.argv) > 2 else (16384, 1024)
x = ops.from_numpy(np.random.default_rng(0).standard_normal((n, l)), torch.device("cuda", 0))
def run():
    qr = ops.QR(x.clone()); return qr.q()
run(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); run(); e1.record(); torch.cuda.synchronize()
print(f"geqrf+orgqr {n}x{l}: {e0.elapsed_time(e1):.2f} ms")
