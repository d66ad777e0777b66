#!/usr/bin/env python3
"""Per-source-line summary of an ncu report (instructions executed, stall samples,
excess shared-memory wavefronts): python tools/ncu_lines.py report.ncu-rep [top]."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, agg = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if hdr is None or r[0] == "" or len(r) < 8:
        continue
    try:
        ins = int(r[hdr["Instructions Executed"]] or 0)
        st = int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        ex = int(r[hdr["L1 Wavefronts Shared Excessive"]] or 0)
    except (ValueError, KeyError):
        continue
    agg.append((fname, int(r[0]), r[1].strip(), ins, st, ex))
ti = sum(a[3] for a in agg) or 1
ts = sum(a[4] for a in agg) or 1
te = sum(a[5] for a in agg) or 1
print(f"instr={ti} samples={ts} smem_excess={te}")
for a in sorted(agg, key=lambda a: -(a[3] / ti + a[4] / ts))[:top]:
    print(f"{a[0][:14]:14s}:{a[1]:<5d} ins {a[3]/ti*100:5.1f}% stall {a[4]/ts*100:5.1f}% bank {a[5]/te*100:5.1f}%  {a[2][:80]}")
