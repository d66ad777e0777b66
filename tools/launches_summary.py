#!/usr/bin/env python
"""Summarise an ncu --csv launch list (one row per metric) into one line per launch."""
import csv
import sys
from collections import OrderedDict

def load(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    hdr, rows = rows[0], rows[1:]
    ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Grid Size", "Block Size", "Metric Name", "Metric Value")}
    out = OrderedDict()
    for r in rows:
        d = out.setdefault(r[ix["ID"]], {"name": r[ix["Kernel Name"]], "grid": r[ix["Grid Size"]], "block": r[ix["Block Size"]]})
        try:
            d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
        except ValueError:
            d[r[ix["Metric Name"]]] = r[ix["Metric Value"]]
    return out

if __name__ == "__main__":
    out = load(sys.argv[1])
    first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    last = int(sys.argv[3]) if len(sys.argv) > 3 else 10**9
    tot = 0.0
    for k, d in out.items():
        if not (first <= int(k) <= last):
            continue
        t = d.get("gpu__time_duration.sum", 0) / 1e3
        tot += t
        rd = d.get("dram__bytes_read.sum", 0) / 1e9
        wr = d.get("dram__bytes_write.sum", 0) / 1e9
        bw = (rd + wr) / (t / 1e6) if t else 0
        print(f"{k:>4} {t:10.1f}us R{rd:7.3f}GB W{wr:7.3f}GB {bw:7.0f}GB/s warps{d.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):6.1f}% {d['grid']:>14} {d['name'][:70]}")
    print(f"total {tot:.1f} us")
