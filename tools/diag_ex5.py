import os, sys, json
sys.path.insert(0, '/root/repo')
import numpy as np, torch
os.environ.setdefault("X", "1")
import paper_2002_07138_b200 as P
from paper_2002_07138_b200 import ops, rangefinder
BL = np.load('/root/repo/tests/golden/baselines.npz')
a = BL["ex5_a"]
orig_add = rangefinder.RankChecks.add
def add(self, count, requested):
    print("check", int(count.item()), requested)
    orig_add(self, count, requested)
rangefinder.RankChecks.add = add
try:
    f = P.randlu(a, 8, q_os=4, p=1, seed=0)
    print("ok", f.p[:5])
except Exception as e:
    print("ERR", e)
