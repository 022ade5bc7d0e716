"""Out-of-core single pass: single_pass_lu over an .rlm file (pinned pipeline,
reader thread + copy stream) vs the HBM-resident DeviceColumnStream on the
same matrix; prints wall times and the file stream's effective GB/s.
usage: python tools/oocore_bench.py [m] [n] [k] [q_os] [panel] [path]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2002_07138_b200 as P

m, n, k, q, panel = (int(x) for x in (sys.argv[1:6] if len(sys.argv) > 5 else (20000, 20000, 360, 360, 1024)))
path = sys.argv[6] if len(sys.argv) > 6 else "/tmp/rlra_oocore.rlm"
rng = np.random.default_rng(0)
x = np.linalg.qr(rng.standard_normal((m, 300)))[0]
y = np.linalg.qr(rng.standard_normal((n, 300)))[0]
a = np.asfortranarray((x * np.arange(1, 301) ** -1.5) @ y.T + 1e-6 * rng.standard_normal((m, n)))
t0 = time.perf_counter()
P.write_rlra(path, a)
print(f"wrote {path}: {8 * m * n / 1e9:.2f} GB in {time.perf_counter() - t0:.1f} s", flush=True)


def timed(fn, reps=2):
    best = 1e30
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        f = fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best, f


dm = P.DeviceMatrix(a)
td, fd = timed(lambda: P.single_pass_lu(P.DeviceColumnStream(dm), k, 0, q_os=q, panel=panel).to_numpy())
tf, ff = timed(lambda: P.single_pass_lu(P.RlraFileColumnStream(path), k, 0, q_os=q, panel=panel))
th, fh = timed(lambda: P.single_pass_lu(P.DenseColumnStream(a), k, 0, q_os=q, panel=panel))
same = np.array_equal(fd.p, ff.p) and np.array_equal(fd.q, ff.q) and np.array_equal(fd.p, fh.p)
print(f"device-resident {td * 1e3:.1f} ms | file stream {tf * 1e3:.1f} ms ({8 * m * n / tf / 1e9:.1f} GB/s) | "
      f"host ndarray stream {th * 1e3:.1f} ms ({8 * m * n / th / 1e9:.1f} GB/s) | pivots identical {same}")
os.remove(path)
