import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2002_07138_b200 import core
dev = torch.device("cuda", 0)
for n in (4_400_000, 50000 * 720, 262144 * 544):
    core.device_gaussian_flat(0, n, dev); torch.cuda.synchronize()
    t0 = time.perf_counter(); x = core.device_gaussian_flat(0, n, dev); torch.cuda.synchronize(); t1 = time.perf_counter()
    t2 = time.perf_counter(); y = np.random.default_rng(0).standard_normal(n); t3 = time.perf_counter()
    print(f"N={n}: device {1e3*(t1-t0):.2f} ms, host numpy {1e3*(t3-t2):.1f} ms, equal={np.array_equal(x.cpu().numpy(), y)}")
