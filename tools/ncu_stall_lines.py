#!/usr/bin/env python3
"""Top source lines for one stall reason from an ncu source dump
(ncu -i rep --page source --csv --print-source cuda,sass [| gzip]):
python tools/ncu_stall_lines.py dump.csv[.gz] stall_long_sb [top]"""
import csv, gzip, io, sys
path, reason = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
txt = (gzip.open(path, "rt") if path.endswith(".gz") else open(path)).read()
fname, hdr, agg = None, None, {}
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}; continue
    if hdr is None or reason not in hdr:
        continue
    if r[0] != "" and not r[0].isdigit():
        continue
    if r[0] != "":  # a CUDA source line: its SASS rows follow
        cur = (fname, int(r[0]), r[1].strip()[:90])
        continue
    if hdr[reason] >= len(r):
        continue
    try:
        v = float(r[hdr[reason]] or 0)
    except ValueError:
        continue
    agg[cur] = agg.get(cur, 0) + v
tot = sum(agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{v / tot * 100:5.1f}%  {k[0]}:{k[1]}  {k[2]}")
