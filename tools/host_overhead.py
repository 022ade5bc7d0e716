"""Host-side (Python) time of one C2 powerlu call with the GPU kept busy
(cProfile, cumulative), to find the call-start latency that shows up as GPU
idle between steps (tools/gap_probe.py)."""
import cProfile
import os
import pstats
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2002_07138_b200 as P  # noqa: E402
from paper_2002_07138_b200 import configs  # noqa: E402

dev = torch.device("cuda", 0)
dm = P.DeviceMatrix(configs.gen_device("C2", dev), 0)
P.set_omega_cache(True)
for _ in range(3):
    P.powerlu(dm, 200, 20, 4, 0)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    P.powerlu(dm, 200, 20, 4, 0)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(45)
st.sort_stats("tottime").print_stats(25)
