"""Aggregate an `ncu --page source --csv --print-source sass,cuda` dump by CUDA
source line: instructions executed and warp-stall samples."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
cur_line = None; cur_file = None; hdr = None
agg = {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; ie = hdr.index("Instructions Executed"); ist = hdr.index("Warp Stall Sampling (All Samples)"); continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0] != "":
        cur_line = (cur_file, int(r[0]), r[1].strip()[:90]); continue
    try:
        e = float(r[ie] or 0); st = float(r[ist] or 0)
    except ValueError:
        continue
    a = agg.setdefault(cur_line, [0.0, 0.0]); a[0] += e; a[1] += st
te = sum(v[0] for v in agg.values()) or 1; ts = sum(v[1] for v in agg.values()) or 1
key = 1 if len(sys.argv) > 2 and sys.argv[2] == "stall" else 0
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
print(f"total warp-instr {te:.3g}, stall samples {ts:.3g}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][key])[:n]:
    print(f"exec {100*v[0]/te:5.1f}%  stall {100*v[1]/ts:5.1f}%  {k[0]}:{k[1]} {k[2]}")
