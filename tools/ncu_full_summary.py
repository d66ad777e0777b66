#!/usr/bin/env python3
"""One line per kernel from `ncu --set full` raw CSV exports (ncu -i rep --page raw --csv):
python tools/ncu_full_summary.py raw1.csv [raw2.csv ...]"""
import csv
import sys


SCALE = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6, "s": 1e3, "second": 1e3,
         "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3}
UNITS = {}


def f(d, k):
    """Value of metric k in ms (times) / GB (bytes) / as exported (others)."""
    try:
        x = float(str(d.get(k, "nan")).replace(",", ""))
    except ValueError:
        return float("nan")
    return x * SCALE.get(UNITS.get(k, ""), 1.0)


print("kernel | ms | DRAM GB/s | DRAM GB (R+W) | L2 hit % | L1TEX/smem lsu wavefronts % | smem wavefronts/SM-cycle | "
      "shared-atomic warp instr | warps active % | regs | IPC | top stalls")
for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    h, v = rows[0], rows[2]
    UNITS.clear()
    UNITS.update(zip(h, rows[1]))
    d = dict(zip(h, v))
    ms = f(d, "gpu__time_duration.sum")  # ms in the raw page
    gb = (f(d, "dram__bytes_read.sum") + f(d, "dram__bytes_write.sum"))
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): f(d, k) for k in h
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    tot = sum(x for x in st.values() if x == x) or 1
    top = ", ".join(f"{k} {100 * x / tot:.0f}%" for k, x in sorted(st.items(), key=lambda kv: -(kv[1] if kv[1] == kv[1] else 0))[:3])
    wf = f(d, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum") / max(f(d, "sm__cycles_elapsed.avg"), 1) / 148
    print(f"{d.get('Kernel Name', '?')[:48]} | {ms:.3f} | {gb / ms * 1e3:.0f} | {gb:.3f} | {f(d, 'lts__t_sector_hit_rate.pct'):.1f} | "
          f"{f(d, 'l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed'):.1f} | {wf:.2f} | "
          f"{f(d, 'smsp__inst_executed_op_shared_atom.sum'):.3g} | {f(d, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | "
          f"{f(d, 'launch__registers_per_thread'):.0f} | {f(d, 'sm__inst_executed.avg.per_cycle_active'):.2f} | {top}")
