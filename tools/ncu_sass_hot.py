"""Summarise an ncu --page source --csv (SASS) dump: hottest instructions by
warp-stall samples and instruction counts."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, ist, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
data = []
for k, r in enumerate(rows[2:]):
    if len(r) != len(hdr) or r[ia] == "Address":
        continue
    data.append((k, float(r[ist] or 0), float(r[iex] or 0), r[isrc].strip()))
ts = sum(d[1] for d in data) or 1
te = sum(d[2] for d in data) or 1
print(f"total stall samples {ts:.0f}, warp-instructions executed {te:.3g}")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for d in sorted(data, key=lambda x: -x[1])[:n]:
    print(f"{d[0]:5d} stall {100*d[1]/ts:5.1f}%  exec {100*d[2]/te:5.1f}%  {d[3][:90]}")
