"""gemm_i8_kernel alone (native per-kernel CUDA-event timer) for the pass shapes
of the BASELINE configs: ms per launch, residue GB/s, int8 TOPS.
usage: python tools/oz_gemm_time.py [shape ...]   shape = m,n,ncols (default: C2 / C3 / C5-block shapes)
RLRA_B200_LIB=<path> picks an alternative build of the library (A/B runs)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2002_07138_b200 import _native, ops

NAMES = ("oz_gemm_i8", "oz_residue_a", "oz_norms", "oz_crt", "oz_residue_b")


def read(lib, name):
    ms, cnt = ctypes.c_double(0.0), ctypes.c_longlong(0)
    lib.rlra_b200_ktimer_read(name.encode(), ctypes.byref(ms), ctypes.byref(cnt))
    return ms.value, cnt.value


shapes = [tuple(int(x) for x in s.split(",")) for s in sys.argv[1:]] or [
    (20000, 10000, 220), (20000, 10000, 200), (16384, 16384, 1024), (50000, 8192, 720), (65536, 32768, 544)]
dev = torch.device("cuda", 0)
lib = _native.load()
for m, n, ncols in shapes:
    a = torch.randn(n, m, dtype=torch.float64, device=dev).t()
    prep = ops.OzPrep(a)
    for trans in (False, True):
        b = torch.randn(ncols, m if trans else n, dtype=torch.float64, device=dev).t()
        for _ in range(2):
            prep.gemm(b, trans=trans)
        torch.cuda.synchronize()
        for nm in NAMES:
            read(lib, nm)
        lib.rlra_b200_ktimer_enable(1)
        for _ in range(5):
            prep.gemm(b, trans=trans)
        torch.cuda.synchronize()
        lib.rlra_b200_ktimer_enable(0)
        ms, cnt = read(lib, "oz_gemm_i8")
        per = ms / max(cnt, 1)
        print(f"{m}x{n} w={ncols} {'TN' if trans else 'NN'}: gemm_i8 {per:8.4f} ms/launch ({cnt} launches)  "
              f"residues {14 * m * n / per / 1e6:7.0f} GB/s  int8 {2 * 14 * m * n * ncols / per / 1e9:7.0f} TOPS",
              flush=True)
    del prep, a
    torch.cuda.empty_cache()
