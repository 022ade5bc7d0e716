"""Pass GEMM (ops.OzPrep) time vs the number of skinny columns: CUDA events
around each product, achieved residue bandwidth nmod*(m*n)/t.
usage: python tools/oz_ncols_bench.py [m] [n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2002_07138_b200 import ops

m = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
n = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
dev = torch.device("cuda", 0)
a = torch.randn(n, m, dtype=torch.float64, device=dev).t()
prep = ops.OzPrep(a)
for ncols in [128, 220, 256, 288, 384, 512, 544, 768, 1024]:
    for trans in (False, True):
        b = torch.randn(ncols, m if trans else n, dtype=torch.float64, device=dev).t()
        prep.gemm(b, trans=trans)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            prep.gemm(b, trans=trans)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"ncols {ncols:5d} {'TN' if trans else 'NN'} {ms:8.3f} ms  residues {14 * m * n / ms / 1e6:7.0f} GB/s", flush=True)
