"""Summarise an ncu --csv launch list (gpu__time_duration.sum per kernel).
usage: python tools/launches.py launches.csv [--last-fraction 0.5]"""
import collections
import csv
import io
import sys


def load(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    seq = []
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        u = r["Metric Unit"]
        v = v / 1e3 if u in ("ns", "nsecond") else (v * 1e3 if u in ("ms", "msecond") else v)
        seq.append((int(r["ID"]), r["Kernel Name"], r["Grid Size"], r["Block Size"], v))
    return seq


def summarise(seq):
    agg = collections.defaultdict(lambda: [0.0, 0])
    for _, name, grid, blk, v in seq:
        short = name.split("(")[0].replace("void ", "")
        agg[short][0] += v
        agg[short][1] += 1
    tot = sum(a[0] for a in agg.values())
    out = []
    for k, (t, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        out.append(f"{t:10.1f} us {100 * t / tot:5.1f}% {c:5d}  {k}")
    out.append(f"{tot:10.1f} us total, {len(seq)} launches")
    return "\n".join(out)


if __name__ == "__main__":
    seq = load(sys.argv[1])
    frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
    print(summarise(seq[int(len(seq) * (1 - frac)):]))
