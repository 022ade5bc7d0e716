"""Constants for the device Gaussian generator: NumPy's PCG64 state for a seed
and the 256-layer ziggurat tables that ``Generator.standard_normal`` uses.

Omega must be bit-identical to the reference's host draw
``np.random.default_rng(seed).standard_normal(m * n)`` (rlra/core.py:33-48),
so the device generator (csrc/rng.cu) replays NumPy's algorithm: PCG64
(128-bit LCG, XSL-RR output) feeding the Marsaglia-Tsang ziggurat.  The
ziggurat tables are read at run time from the NumPy installation itself (the
`ki_double` / `wi_double` / `fi_double` symbols of numpy/random/_generator),
never copied into this repository, and a host replay of the first draws of a
probe seed must match NumPy exactly before the device generator is enabled.
"""

from __future__ import annotations

import functools
import os
import struct

import numpy as np

PCG64_MULT = 0x2360ED051FC65DA44385DF649FCCF645
ZIGGURAT_NOR_R = 3.6541528853610087963519472518
ZIGGURAT_NOR_INV_R = 0.27366123732975827203338247596
MASK64 = (1 << 64) - 1


def pcg64_state(seed):
    """(state, inc) of np.random.default_rng(seed)'s PCG64 as 128-bit ints."""
    st = np.random.PCG64(seed).state["state"]
    return int(st["state"]), int(st["inc"])


def _elf_symbols(path, names):
    """Minimal ELF64 little-endian reader: file bytes of the named objects."""
    with open(path, "rb") as fh:
        data = fh.read()
    if data[:4] != b"\x7fELF" or data[4] != 2 or data[5] != 1:
        raise ValueError("not an ELF64 LE file")
    e_shoff, = struct.unpack_from("<Q", data, 0x28)
    e_shentsize, e_shnum, e_shstrndx = struct.unpack_from("<HHH", data, 0x3A)
    secs = []
    for i in range(e_shnum):
        off = e_shoff + i * e_shentsize
        (sh_name, sh_type, sh_flags, sh_addr, sh_offset, sh_size, sh_link, sh_info, sh_addralign,
         sh_entsize) = struct.unpack_from("<IIQQQQIIQQ", data, off)
        secs.append((sh_name, sh_type, sh_addr, sh_offset, sh_size, sh_link, sh_entsize))
    out = {}
    for (_, sh_type, _, sh_offset, sh_size, sh_link, sh_entsize) in secs:
        if sh_type != 2:  # SHT_SYMTAB
            continue
        strtab = secs[sh_link]
        for k in range(sh_size // sh_entsize):
            st_name, st_info, st_other, st_shndx, st_value, st_size = struct.unpack_from(
                "<IBBHQQ", data, sh_offset + k * sh_entsize)
            end = data.index(b"\0", strtab[3] + st_name)
            name = data[strtab[3] + st_name:end].decode(errors="replace")
            if name in names and st_shndx < len(secs) and st_size:
                sec = secs[st_shndx]
                foff = sec[3] + (st_value - sec[2])
                out[name] = data[foff:foff + st_size]
    return out


@functools.lru_cache(maxsize=1)
def tables():
    """(ki uint64[256], wi float64[256], fi float64[256]) from NumPy's binary."""
    import numpy.random as npr

    d = os.path.dirname(npr.__file__)
    cands = sorted(f for f in os.listdir(d) if f.startswith("_generator") and f.endswith(".so"))
    if not cands:
        raise RuntimeError("numpy.random._generator extension not found")
    syms = _elf_symbols(os.path.join(d, cands[0]), {"ki_double", "wi_double", "fi_double"})
    if set(syms) != {"ki_double", "wi_double", "fi_double"}:
        raise RuntimeError("ziggurat tables not found in numpy's _generator symbol table")
    ki = np.frombuffer(syms["ki_double"], dtype="<u8").copy()
    wi = np.frombuffer(syms["wi_double"], dtype="<f8").copy()
    fi = np.frombuffer(syms["fi_double"], dtype="<f8").copy()
    if not (ki.shape == wi.shape == fi.shape == (256,)):
        raise RuntimeError("unexpected ziggurat table sizes")
    return ki, wi, fi


def host_replay(seed, count):
    """Pure-Python replay of Generator(PCG64(seed)).standard_normal(count) with
    the extracted tables (validation of the constants; slow, small counts)."""
    ki, wi, fi = tables()
    state, inc = pcg64_state(seed)
    m128 = (1 << 128) - 1

    def next_u64():
        nonlocal state
        state = (state * PCG64_MULT + inc) & m128
        hi, lo = state >> 64, state & MASK64
        x = hi ^ lo
        rot = hi >> 58
        return ((x >> rot) | (x << ((64 - rot) & 63))) & MASK64

    def next_double():
        return (next_u64() >> 11) * (1.0 / 9007199254740992.0)

    out = np.empty(count)
    for i in range(count):
        while True:
            r = next_u64()
            idx = r & 0xFF
            r >>= 8
            sign = r & 1
            rabs = (r >> 1) & 0x000FFFFFFFFFFFFF
            x = rabs * float(wi[idx])
            if sign:
                x = -x
            if rabs < int(ki[idx]):
                out[i] = x
                break
            if idx == 0:
                while True:
                    xx = -ZIGGURAT_NOR_INV_R * np.log1p(-next_double())
                    yy = -np.log1p(-next_double())
                    if yy + yy > xx * xx:
                        out[i] = -(ZIGGURAT_NOR_R + xx) if (rabs >> 8) & 1 else ZIGGURAT_NOR_R + xx
                        break
                break
            if (float(fi[idx - 1]) - float(fi[idx])) * next_double() + float(fi[idx]) < np.exp(-0.5 * x * x):
                out[i] = x
                break
    return out


@functools.lru_cache(maxsize=1)
def validated():
    """True when the extracted constants reproduce NumPy on a probe seed."""
    try:
        ref = np.random.default_rng(12345).standard_normal(4000)
        return bool(np.array_equal(host_replay(12345, 4000), ref))
    except Exception:
        return False
