"""Print the CUDA error a cooperative GEPP launch returns (debug aid under ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2002_07138_b200 import ops
a = ops.as_fmat(torch.randn((220, 10000), dtype=torch.float64, device="cuda").t().clone())
try:
    ops.getrf_(a); torch.cuda.synchronize(); print("getrf ok")
except Exception as e:
    print("getrf error:", e)
