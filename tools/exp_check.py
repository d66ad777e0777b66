"""A/B helper: for each experiment bit set given on the command line, check that
the experiment path produces the product path's output (bit-exact) on C2/C3-
sized device graphs and print the per-level times of both.
Usage: python tools/exp_check.py 64 [128 ...]  [--configs C2,C3] [--steps 10]"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2501_06872_b200 import gen, set_config, transpose_device


def run(off, edg, V, steps):
    acc = [0.0] * 7
    out = None
    for i in range(steps + 2):
        t_off, t_edg, st = transpose_device(off, edg, V, want_stats=True)
        if i >= 2:
            vals = [st.ms_step1, st.ms_step2, st.ms_step3] + [st.ms_kernel[k] for k in range(4)]
            acc = [a + v / steps for a, v in zip(acc, vals)]
        out = (t_off, t_edg)
    return out, acc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("bits", type=int, nargs="+")
    ap.add_argument("--configs", default="C2,C3")
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    for name in a.configs.split(","):
        cfg = gen.CONFIGS[name]
        off, edg = gen.generate_device(cfg, device="cuda")
        V = cfg.num_vertices
        set_config()
        ref, t0 = run(off, edg, V, a.steps)
        print(f"{name} product      L1 {t0[0]:.3f} L2 {t0[1]:.3f} L3 {t0[2]:.3f} sum {sum(t0[:3]):.3f} | "
              f"p1 {t0[3]:.3f} p2 {t0[4]:.3f} p3 {t0[5]:.3f} big {t0[6]:.3f}", flush=True)
        for b in a.bits:
            set_config(experiment=b)
            out, t = run(off, edg, V, a.steps)
            same = bool(torch.equal(out[0], ref[0]) and torch.equal(out[1], ref[1]))
            print(f"{name} experiment {b:4d} L1 {t[0]:.3f} L2 {t[1]:.3f} L3 {t[2]:.3f} sum {sum(t[:3]):.3f} | "
                  f"p1 {t[3]:.3f} p2 {t[4]:.3f} p3 {t[5]:.3f} big {t[6]:.3f} | equal={same}", flush=True)
            del out
        set_config()
        del ref, off, edg
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
