"""Staged check of the Ozaki-II int8 path (csrc/ozaki.cu) on the GPU:
residues of A and B, the int8 tensor-core products mod m_l, the CRT result,
and the final accuracy against an exact (Python-integer) product.

    python tools/oz_check.py [m n l]
"""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_07138_b200 import ops  # noqa: E402

MODS = [249, 247, 245, 244, 241, 239, 233, 229, 227, 223, 211, 199, 197, 193, 191, 181]
T = 128


def unswizzle(tile):
    """16 KB swizzled tile bytes -> (128 rows, 128 bytes) logical."""
    t = tile.reshape(128, 8, 16)
    out = np.empty_like(t)
    for r in range(128):
        for c in range(8):
            out[r, c] = t[r, (c ^ (r & 7))]
    return out.reshape(128, 128)


def budget(nmod):
    lg = sum(math.log2(MODS[l]) for l in range(nmod))
    tot = int(math.floor(lg)) - 2
    return min(55, tot - tot // 2), min(55, tot // 2)


def main():
    m, n, l = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (700, 500, 100)
    nmod = ops.OZ_NMOD
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(1)
    a = rng.standard_normal((m, n))
    a[3, :] *= 1e-3
    a[:, 5] *= 7.0
    ad = ops.from_numpy(a, dev)
    prep = ops.OzPrep(ad, nmod)
    torch.cuda.synchronize()
    ws = prep.ws.cpu().numpy()
    e_a = int(ws[:4].view(np.int32)[0])
    pa, pb = budget(nmod)
    nib = -(-m // T); nib += nib & 1
    njb = -(-n // T); njb += njb & 1
    ncb = -(-n // 256)
    nrb = -(-m // 2048)
    off_tiles = (256 + ncb * m * 8 + nrb * n * 8 + 1023) & ~1023
    print(f"e_a={e_a} pa={pa} pb={pb} nib={nib} njb={njb}")
    x = np.rint(a * 2.0 ** e_a).astype(np.int64)
    maxnorm = max(np.sqrt((a * a).sum(0)).max(), np.sqrt((a * a).sum(1)).max())
    assert maxnorm * 2.0 ** e_a < 2.0 ** pa and maxnorm * 2.0 ** e_a >= 2.0 ** (pa - 1), (maxnorm, e_a)
    xpad = np.zeros((nib * T, njb * T), dtype=np.int64)
    xpad[:m, :n] = x
    bad = 0
    for li in range(nmod):
        mod = MODS[li]
        for jb in range(njb):
            for ib in range(nib):
                off = off_tiles + ((li * njb + jb) * nib + ib) * T * T
                tile = unswizzle(ws[off:off + T * T]).view(np.int8).astype(np.int64)  # [j][i]
                ref = xpad[ib * T:(ib + 1) * T, jb * T:(jb + 1) * T].T
                if not (np.all((tile - ref) % mod == 0) and np.abs(tile).max() <= 127):
                    bad += 1
    print("A residue tiles bad:", bad)

    for trans in (1, 0):
        k, rows = (m, n) if trans else (n, m)
        b = rng.standard_normal((k, l))
        bd = ops.from_numpy(b, dev)
        c, gws = prep.gemm(bd, trans=bool(trans), keep_ws=True)
        torch.cuda.synchronize()
        c = ops.to_numpy(c)
        g = gws.cpu().numpy()
        ng = -(-l // 256); n_g = -(-(-(-l // ng)) // 32) * 32
        cols_pad = ng * n_g
        nkb = nib if trans else njb
        nmb = (njb if trans else nib) // 2
        rows_pad = nmb * 256
        off_b = (cols_pad * 4 + 1023) & ~1023
        off_t = off_b + nmod * cols_pad * nkb * T
        e_b = g[:cols_pad * 4].view(np.int32)[:l].astype(np.int64)
        y = np.rint(b * 2.0 ** e_b[None, :]).astype(np.int64)
        ypad = np.zeros((nkb * T, cols_pad), dtype=np.int64)
        ypad[:k, :l] = y
        bbad = 0
        for li in range(nmod):
            mod = MODS[li]
            for gi in range(ng):
                for kb in range(nkb):
                    off = off_b + ((li * ng + gi) * nkb + kb) * n_g * T
                    tl = g[off:off + n_g * T]
                    t8 = np.stack([unswizzle(np.concatenate([tl[r0 * T:(r0 + 8) * T], np.zeros(T * T - 8 * T, np.uint8)]))[:8]
                                   for r0 in range(0, n_g, 8)]).reshape(n_g, T).view(np.int8).astype(np.int64)
                    ref = ypad[kb * T:(kb + 1) * T, gi * n_g:(gi + 1) * n_g].T
                    if not np.all((t8 - ref) % mod == 0):
                        bbad += 1
        print(f"trans={trans}: B residue tiles bad: {bbad}")
        # integer products mod m from the t array
        xx = (xpad[:m, :n].T if trans else xpad[:m, :n])  # rows x k
        tbad = 0
        big_m = math.prod(MODS[:nmod])
        for li in range(nmod):
            mod = MODS[li]
            ycrt = pow((big_m // mod) % mod, -1, mod)
            xm = (xx % mod).astype(np.int64)
            ym = (y % mod).astype(np.int64)
            ref = ((xm @ ym) % mod * ycrt) % mod  # rows x l, exact in int64
            tt = g[off_t + li * cols_pad * rows_pad: off_t + (li + 1) * cols_pad * rows_pad].reshape(cols_pad, rows_pad)
            got = tt[:l, :rows].T.astype(np.int64)
            nb = int((got != ref).sum())
            if nb:
                tbad += 1
                if tbad <= 2:
                    w = np.argwhere(got != ref)
                    print(f"  modulus {li}: {nb} wrong of {got.size}; first {w[:4].tolist()} got {got[tuple(w[0])]} ref {ref[tuple(w[0])]}")
        print(f"trans={trans}: moduli with wrong products: {tbad}")
        exact = (a.T if trans else a) @ b
        err = np.abs(c - exact).max() / np.abs(exact).max()
        ld = (a.T if trans else a).astype(np.longdouble) @ b.astype(np.longdouble)
        err_ld = float(np.abs(c - ld).max() / np.abs(ld).max())
        err_np = float(np.abs(exact - ld).max() / np.abs(ld).max())
        print(f"trans={trans}: max rel err vs numpy {err:.3e}; vs longdouble: ozaki {err_ld:.3e}  numpy-dgemm {err_np:.3e}")


if __name__ == "__main__":
    main()
