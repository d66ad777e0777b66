"""Group an `ncu --page source --csv --print-source sass,cuda` dump into phases by
(file, line range): usage ncu_phase.py dump.csv file:lo-hi=name ..."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
specs = []
for a in sys.argv[2:]:
    loc, name = a.split("=")
    f, rng = loc.split(":")
    lo, hi = map(int, rng.split("-"))
    specs.append((f, lo, hi, name))
cur = None; hdr = None; agg = {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; ie = hdr.index("Instructions Executed"); ist = hdr.index("Warp Stall Sampling (All Samples)"); continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0] != "":
        cur = (cur_file, int(r[0])); continue
    try:
        e = float(r[ie] or 0); st = float(r[ist] or 0)
    except ValueError:
        continue
    name = "other"
    for f, lo, hi, nm in specs:
        if cur and cur[0] == f and lo <= cur[1] <= hi:
            name = nm; break
    a = agg.setdefault(name, [0.0, 0.0]); a[0] += e; a[1] += st
te = sum(v[0] for v in agg.values()) or 1; ts = sum(v[1] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:12s} exec {100*v[0]/te:5.1f}%  stall {100*v[1]/ts:5.1f}%")
