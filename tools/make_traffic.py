#!/usr/bin/env python
"""Per-step and per-kernel DRAM traffic (ncu dram__bytes_read.sum + write.sum)
from an ncu --csv launch list of `bench.py --steps 1`: the last complete
transpose in the list (launches from one k_set_u32 to the next).
Usage: make_traffic.py launches.csv config [profiles/ncu_traffic.json]; config = C1..C5 or the
workload name bench.py looks up (gen.CONFIGS[...].name)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from launches_summary import load  # noqa: E402

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2501_06872_b200 import gen  # noqa: E402

if sys.argv[2] in gen.CONFIGS:
    sys.argv[2] = gen.CONFIGS[sys.argv[2]].name

out = load(sys.argv[1])
keys = list(out.keys())
starts = [i for i, k in enumerate(keys) if "k_set_u32" in out[k]["name"]]
if len(starts) < 2:
    raise SystemExit("need at least two transposes in the launch list")
a, b = starts[-2], starts[-1]
step = [out[k] for k in keys[a:b]]
tot = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in step)
kern = {}
for d in step:
    n = d["name"]
    key = None
    if "k_p1" in n:
        key = "k_p1"
    elif "k_p2" in n and "DecR1" in n:
        key = "k_p2"
    elif "k_p2" in n and "DecR2" in n:
        key = "k_p2_big"
    elif "k_p3" in n:
        key = "k_p3"
    if key:
        kern[key] = int(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0))
path = Path(sys.argv[3] if len(sys.argv) > 3 else "profiles/ncu_traffic.json")
db = json.loads(path.read_text()) if path.exists() else {}
db[sys.argv[2]] = {"step_bytes": int(tot), "kernels": kern, "source": Path(sys.argv[1]).name,
                   "step_ms_ncu_serialised": sum(d.get("gpu__time_duration.sum", 0) for d in step) / 1e6}
path.write_text(json.dumps(db, indent=1) + "\n")
print(sys.argv[2], db[sys.argv[2]])
