#!/usr/bin/env python
"""Benchmark: CSR->CSC transposition edges/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

N=1: the workload is config C3 (RMAT scale 24, edge factor 32, IDs permuted:
|V| = 2^24, |E| = 2^29), the north_star's single-GPU target.  The graph is
generated on the device with the package's seeded generator (synthetic data; the
paper's datasets are not available).  A step = one full transpose (every
kernel) of the device-resident CSR; inputs (2.3 GB) exceed the 126 MB L2, so no
flush is needed between steps.  Timing: CUDA events on the launching stream,
barrier + synchronize on both sides, max over ranks.

N>1 (torchrun, one process per GPU, NCCL): each rank owns an edge-balanced
source shard of the same graph; a step = sender partition + NCCL all-to-all of
records + receiver transpose of its destination range (strong scaling).

--impl reference: the reference's CPU algorithms on the box's host cores, as
OpenMP ports (oracle/gt_oracle.c): transpose_scantrans (baselines.py:265-312),
transpose_atomic + sort_neighbor_lists (baselines.py:168-209, 457-475) and
transpose_potra (hlh.py:441-588) + sort_neighbor_lists; the timed steps run the
fastest of them.  The input graph is generated on the host by oracle/ (same
seeded draws as gen.py), so this arm never loads the product library.  The
reference itself is Python + numba and is not installed on the GPU box.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "CSR→CSC edges/sec at 1/2/4/8 B200; achieved HBM GB/s vs peak"
FALLBACK_HBM = 6650.0


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def algo_bytes(V: int, E: int) -> int:
    """north_star roofline bytes: offsets + neighbours read for both passes,
    CSC written = 2*(8(V+1) + 4E) + (8(V+1) + 4E) = 24(V+1) + 12E."""
    return 24 * (V + 1) + 12 * E


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the timed region runs."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int = 0, period_ms: int = 50):
        self.path = tempfile.mktemp(suffix=".csv")
        self.proc = None
        self.gpu = gpu_index
        self.period = period_ms

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 f"-lms={self.period}"], stdout=self.f, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.15)
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in Path(self.path).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.path)
        return {
            "sm_mhz": statistics.median(sm) if sm else None,
            "sm_max_mhz": max(smax) if smax else None,
            "reasons": sorted(reasons),
            "samples": len(sm),
        }


def cpu_scantrans(off: np.ndarray, edg: np.ndarray, V: int, threads: int, reps: int):
    from oracle import oracle

    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        oracle.transpose_scantrans_c(off, edg, V, threads)
        times.append(time.perf_counter() - t0)
    return times


# The reference's CPU paths that produce this path's output (CSC, lists ascending by
# source), as OpenMP ports in oracle/gt_oracle.c (test infrastructure; the reference is
# Python + numba and is not installed on the GPU box):
#   scantrans     transpose_scantrans (baselines.py:265-312), sorted by construction
#   atomic+sort   transpose_atomic (baselines.py:168-209) + sort_neighbor_lists (457-475)
#   potra+sort    transpose_potra auto: step 0 sample/probe, HLH steps 1-3 or the atomic
#                 delegate (hlh.py:441-588) + sort_neighbor_lists
def cpu_path(name: str, off, edg, V: int, threads: int):
    """Run one reference CPU path once: (seconds, per-phase seconds)."""
    from oracle import oracle

    t0 = time.perf_counter()
    if name == "scantrans":
        oracle.transpose_scantrans_c(off, edg, V, threads)
        return time.perf_counter() - t0, {}
    if name == "atomic+sort":
        lib = oracle.load()
        o = np.ascontiguousarray(off, dtype=np.uint64)
        e = np.ascontiguousarray(edg, dtype=np.uint32)
        to = np.empty(V + 1, np.uint64)
        te = np.empty(e.shape[0], np.uint32)
        oracle._check(lib.gto_transpose_atomic(oracle._p(o), oracle._p(e), V, e.shape[0], oracle._p(to),
                                               oracle._p(te), threads, 1 << 18), "atomic")
        t1 = time.perf_counter()
        oracle._check(lib.gto_sort_lists(oracle._p(to), V, oracle._p(te), threads), "sort")
        t2 = time.perf_counter()
        return t2 - t0, {"steps1-3": t1 - t0, "sort": t2 - t1}
    if name == "potra+sort":
        _, _, info = oracle.transpose_potra_c(off, edg, V, threads, sort=True)
        ph = {k: float(v) for k, v in info["phase_times"].items()}
        ph["method_chosen"] = info["method_chosen"]
        ph["k"] = info["k"]
        return time.perf_counter() - t0, ph
    raise ValueError(name)


CPU_PATHS = ("scantrans", "atomic+sort", "potra+sort")


def cpu_paths_report(off, edg, V: int, threads: int, budget_s: float):
    """Each reference CPU path once on a bounded sample of the workload (a source
    prefix sized so that all paths together take about budget_s).  Returns
    (report dict, fastest path name, sample arrays, sample description)."""
    E = int(off[-1])
    p_off, p_edg, _ = source_prefix_sample(off, edg, 1 << 24)
    t_probe, _ = cpu_path("scantrans", p_off, p_edg, V, threads)
    per_edge = t_probe / max(int(p_off[-1]), 1)
    target = int(budget_s / max(per_edge * 3.0, 1e-12))
    s_off, s_edg, desc = source_prefix_sample(off, edg, max(target, 1 << 20))
    Es = int(s_off[-1])
    rep = {}
    for name in CPU_PATHS:
        secs, ph = cpu_path(name, s_off, s_edg, V, threads)
        rep[name] = {"edges_per_s": Es / secs, "seconds": secs, "phases": ph}
    best = max(rep, key=lambda n: rep[n]["edges_per_s"])
    return rep, best, (s_off, s_edg), desc


def source_prefix_sample(off: np.ndarray, edg: np.ndarray, max_edges: int):
    """Bounded sample of the workload: the smallest source prefix holding
    >= max_edges edges (its full out-lists; destinations span all of V)."""
    E = int(off[-1])
    if E <= max_edges:
        return off, edg, "full graph"
    s = int(np.searchsorted(off, np.uint64(max_edges), side="left"))
    sub_off = off[: s + 1].copy()
    V = off.shape[0] - 1
    full_off = np.concatenate([sub_off, np.full(V - s, sub_off[-1], dtype=np.uint64)])
    return full_off, edg[: int(sub_off[-1])], f"source prefix [0,{s}) with {int(sub_off[-1])} edges"


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args, cfg, rank: int):
    """--impl reference: the reference's CPU paths (OpenMP ports) on the host cores.
    The input graph is generated on the host by the oracle library (the same seeded
    draws as gen.py): this process never loads the product library."""
    if rank != 0:
        return
    from oracle import oracle

    oracle.load()
    threads = host_cores()
    V = cfg.num_vertices
    if cfg.kind in ("rmat", "er"):
        off, edg = oracle.generate_c(cfg, threads)
    else:
        from paper_2501_06872_b200 import gen  # numpy generator (no native library)

        off, edg = gen.generate_np(cfg)
    E = int(off[-1])
    steps, warm = max(1, args.steps), max(0, args.warmup)
    # warm-up = one run of every path on a bounded sample (also picks the fastest
    # sorted path); each timed step = one run of that path on the same sample
    rep, best, (s_off, s_edg), desc = cpu_paths_report(off, edg, V, threads, 20.0)
    per = rep[best]["seconds"]
    if per * (steps + warm) > 150.0:  # shrink the sample so the whole run ends in minutes
        target = int(int(s_off[-1]) * 150.0 / (per * (steps + warm)))
        s_off, s_edg, desc = source_prefix_sample(off, edg, max(target, 1 << 20))
    for _ in range(max(0, warm - 1)):
        cpu_path(best, s_off, s_edg, V, threads)
    times = [cpu_path(best, s_off, s_edg, V, threads)[0] for _ in range(steps)]
    Es = int(s_off[-1])
    total = sum(times)
    value = Es * len(times) / total
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": "edges/s",
        "n_gpus": args.gpus,
        "steps": steps,
        "warmup": warm,
        "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u32",
        "data": "synthetic",
        "config": {"workload": cfg.name, "num_vertices": V, "num_edges": E, "sample_edges": Es},
        "cpu_baseline": {"value": value, "unit": "edges/s", "cores": threads, "kind": "port",
                         "sample": f"{desc}; fastest sorted reference path = {best} (OpenMP port, "
                                   "oracle/gt_oracle.c); input generated on the host by oracle/",
                         "paths": rep},
        "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--force-dist", action="store_true", help="use the sharded path even at N=1")
    ap.add_argument("--no-graph", action="store_true", help="time plain launches instead of CUDA-graph replays")
    ap.add_argument("--capi", action="store_true",
                    help="sharded runs: also time the step as one gt_transpose_multi (C ABI, NCCL from libgt.so) call")
    ap.add_argument("--experiment", type=int, default=0, help="A/B experiment bits (gt_config.reserved[0]); 0 = product")
    ap.add_argument("--rank-mode", type=int, default=-1, help="-1 auto, 0 smem-atomic, 1 safe OR-mask ranking")
    ap.add_argument("--split", default=None, help="experiment: digit split a,b,c (gt_config.split)")
    ap.add_argument("--force-wide", action="store_true", help="experiment: the wide form (gt_config.force_wide)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3  # timing rule: >= 3 warm-up steps

    from paper_2501_06872_b200 import gen

    cfg = gen.CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, cfg, rank)
        return

    import torch

    torch.cuda.set_device(local_rank)
    dist_on = world > 1 or args.force_dist
    if dist_on:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local_rank))

    from paper_2501_06872_b200 import _lib, set_config, set_rank_mode, transpose_device

    if args.experiment or args.split or args.force_wide:
        set_config(split=tuple(int(x) for x in args.split.split(",")) if args.split else None,
                   force_wide=args.force_wide, experiment=args.experiment)
    if args.rank_mode >= 0:
        set_rank_mode(args.rank_mode)

    V = cfg.num_vertices
    dev = torch.device("cuda", local_rank)
    off_d, edg_d = gen.generate_device(cfg, device=dev)
    E = int(edg_d.numel())
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    peak, peak_src = _peaks()
    sampler = ClockSampler(local_rank)

    e2e_dist = None
    if not dist_on:
        t_off = torch.empty(V + 1, dtype=torch.int64, device=dev)
        t_edg = torch.empty(E, dtype=torch.int32, device=dev)
        from paper_2501_06872_b200 import transpose_status

        s = torch.cuda.Stream(device=dev)
        stream = s
        with torch.cuda.stream(s):
            for _ in range(args.warmup):
                transpose_device(off_d, edg_d, V, t_offsets=t_off, t_edges=t_edg, stream=s)
        s.synchronize()
        graph = None
        if not args.no_graph:
            # the whole transpose (every kernel, the side-stream fork/join included) as one CUDA
            # graph: replays carry no host launch gaps; the work per replay is the full step
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=s):
                transpose_device(off_d, edg_d, V, t_offsets=t_off, t_edges=t_edg, stream=s)
            with torch.cuda.stream(s):
                graph.replay()
            s.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sampler.start()
        torch.cuda.synchronize()
        with torch.cuda.stream(s):  # graph replays launch on the current stream
            ev0.record(s)
            for _ in range(args.steps):
                if graph is not None:
                    graph.replay()
                else:
                    transpose_device(off_d, edg_d, V, t_offsets=t_off, t_edges=t_edg, stream=s)
            ev1.record(s)
        torch.cuda.synchronize()
        clocks = sampler.stop()
        transpose_status(stream=s)
        ms = ev0.elapsed_time(ev1) / args.steps
        # per-level and per-kernel CUDA events of the library (gt_stats), from the same number of
        # steps run right after the timed region (each such call waits for its events)
        acc = {"step1": 0.0, "step2": 0.0, "step3": 0.0, "k": [0.0, 0.0, 0.0, 0.0]}
        for _ in range(args.steps):
            _, _, st = transpose_device(off_d, edg_d, V, t_offsets=t_off, t_edges=t_edg, want_stats=True)
            acc["step1"] += st.ms_step1
            acc["step2"] += st.ms_step2
            acc["step3"] += st.ms_step3
            for i in range(4):
                acc["k"][i] += st.ms_kernel[i]
        launches = int(st.n_launches) * args.steps
        K = args.steps
        kern = {"step1_ms": acc["step1"] / K, "step2_ms": acc["step2"] / K, "step3_ms": acc["step3"] / K,
                "digit_bits": list(st.bits), "big_buckets": int(st.n_big_buckets),
                "rank_mode": "smem-atomic" if st.rank_mode == 0 else "or-mask",
                "workspace_bytes": int(st.workspace_bytes),
                "timed_region": "CUDA-graph replays of the whole transpose" if graph is not None
                                else "plain launches of the whole transpose"}
        kernel_ms = [x / K for x in acc["k"]]
        n_gpus = 1
    else:
        import torch.distributed as dist

        from paper_2501_06872_b200.multi import GpuShardBackend, distributed_step, plan_shards, shard_geometry

        off_h = off_d.cpu().numpy().view(np.uint64)
        plan = plan_shards(off_h, world)
        geom = shard_geometry(V, E)
        e0, e1 = int(plan.edge_bounds[rank]), int(plan.edge_bounds[rank + 1])
        edg_slice = edg_d[e0:e1].clone()
        del edg_d
        torch.cuda.empty_cache()
        backend = GpuShardBackend(dev)

        def dstep(timings=None, check=True):
            return distributed_step(off_d, edg_slice, V, E, plan, rank, backend, geom=geom, timings=timings,
                                    check_status=check)

        for _ in range(args.warmup):
            dstep()
        torch.cuda.synchronize()
        dist.barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sampler.start()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            dstep(check=False)  # the overflow status is read once after the timed region
        ev1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        clocks = sampler.stop()
        from paper_2501_06872_b200 import transpose_status

        transpose_status(device=dev)
        t = torch.tensor([ev0.elapsed_time(ev1)], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item()) / args.steps
        # per-phase device times (CUDA events inside the step; max over ranks), after the timed region
        ph = {"send_ms": 0.0, "exchange_ms": 0.0, "receive_ms": 0.0}
        nph = max(1, min(args.steps, 5))
        tim = {}
        for _ in range(nph):
            tim = {}
            dstep(tim)
            for k in ph:
                ph[k] += tim[k] / nph
        pt = torch.tensor([ph["send_ms"], ph["exchange_ms"], ph["receive_ms"]], device=dev, dtype=torch.float64)
        dist.all_reduce(pt, op=dist.ReduceOp.MAX)
        # our kernels per step: sender level 1 (tile owners x2, count-tile owners, count, scan, place, meta)
        # + receiver (gt_stats.n_launches); NCCL's own kernels are not counted
        launches = (7 + int(tim.get("receive_launches") or 0)) * args.steps
        kern = {"src_bounds": plan.src_bounds.tolist(), "bucket_range": list(tim.get("buckets", ())),
                "records_received": tim.get("records_received"),
                "phases_ms_max_over_ranks": {"send (level 1)": float(pt[0]), "exchange (count all-gather + "
                                             "NCCL all-to-all of R1, 4 B/edge)": float(pt[1]),
                                             "receive (levels 2-3)": float(pt[2])},
                "bytes_on_wire_per_edge": 4}
        if args.capi:
            # the same step as one C-ABI call per rank (gt_transpose_multi: NCCL driven from
            # libgt.so); its slice must equal the torch.distributed orchestration's
            from paper_2501_06872_b200.multi import MultiComm

            def bcast(b):
                obj = [b]
                dist.broadcast_object_list(obj, src=0)
                return obj[0]

            comm = MultiComm(rank, world, broadcast=bcast)
            src0, src1 = int(plan.src_bounds[rank]), int(plan.src_bounds[rank + 1])
            cap = int(1.1 * E / world) + (1 << 20)
            to_c, te_c, info = comm.transpose(off_d, edg_slice, V, E, src0, src1, capacity=cap)
            to_p, te_p, _, _ = dstep()
            same = bool(torch.equal(to_c, to_p) and torch.equal(te_c, te_p))
            torch.cuda.synchronize()
            dist.barrier()
            e0c, e1c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            nc = max(3, min(args.steps, 10))
            e0c.record(stream)
            for _ in range(nc):
                comm.transpose(off_d, edg_slice, V, E, src0, src1, capacity=cap)
            e1c.record(stream)
            torch.cuda.synchronize()
            tc = torch.tensor([e0c.elapsed_time(e1c) / nc, info.ms_send, info.ms_exchange, info.ms_receive],
                              device=dev, dtype=torch.float64)
            dist.all_reduce(tc, op=dist.ReduceOp.MAX)
            okt = torch.tensor([1 if same else 0], device=dev)
            dist.all_reduce(okt, op=dist.ReduceOp.MIN)
            kern["c_abi_gt_transpose_multi"] = {"ms_per_step": float(tc[0]), "send_ms": float(tc[1]),
                                                "exchange_ms": float(tc[2]), "receive_ms": float(tc[3]),
                                                "equals_torch_distributed_step": bool(okt.item()),
                                                "steps": nc}
            comm.close()
        n_gpus = world
        e2e_dist = None
        if not args.no_e2e:
            # end to end per rank: H2D of the offsets and this rank's edge slice from pinned
            # host memory, the sharded step, D2H of this rank's CSC slice into pinned memory;
            # CUDA events on the launching stream (the copies are on it), max over ranks
            h_off = off_d.cpu().pin_memory()
            h_edg = edg_slice.cpu().pin_memory()
            t_off_s, t_edg_s, _, _ = dstep()
            h_toff = torch.empty(t_off_s.shape, dtype=t_off_s.dtype).pin_memory()
            h_tedg = torch.empty(t_edg_s.shape, dtype=t_edg_s.dtype).pin_memory()

            def e2e_step():
                off_d.copy_(h_off, non_blocking=True)
                edg_slice.copy_(h_edg, non_blocking=True)
                to, te, _, _ = dstep()
                h_toff.copy_(to, non_blocking=True)
                h_tedg.copy_(te, non_blocking=True)

            e2e_step()
            torch.cuda.synchronize()
            dist.barrier()
            ne = max(3, min(args.steps, 10))
            e0v, e1v = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0v.record(stream)
            for _ in range(ne):
                e2e_step()
            e1v.record(stream)
            torch.cuda.synchronize()
            dist.barrier()
            te_ms = torch.tensor([e0v.elapsed_time(e1v) / ne], device=dev, dtype=torch.float64)
            dist.all_reduce(te_ms, op=dist.ReduceOp.MAX)
            nb = torch.tensor([h_off.numel() * 8 + h_edg.numel() * 4, h_toff.numel() * 8 + h_tedg.numel() * 4],
                              device=dev, dtype=torch.int64)
            dist.all_reduce(nb)  # whole-job bytes per step
            te = float(te_ms.item()) / 1e3
            e2e_dist = {"value": E / te, "unit": "edges/s", "h2d_bytes_per_step": int(nb[0]),
                        "d2h_bytes_per_step": int(nb[1]), "ms_per_step": te * 1e3, "steps": ne,
                        "api": "per rank: pinned H2D of offsets + its edge slice, distributed_step "
                               "(multi.py), pinned D2H of its CSC slice; max over ranks"}

    value = E / (ms / 1e3)
    abytes = algo_bytes(V, E)
    achieved = abytes / (ms / 1e3) / 1e9
    agg_peak = peak * n_gpus
    traffic, ktraffic = None, {}
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists() and not dist_on:  # the ncu table describes the single-GPU pipeline only
        try:
            tj = json.loads(tf.read_text()).get(cfg.name) or {}
            traffic = tj.get("step_bytes")
            ktraffic = tj.get("kernels", {})
        except Exception:
            traffic, ktraffic = None, {}
    if not dist_on:
        # per-kernel roofline: algorithmic bytes of each main kernel over its
        # CUDA-event time inside the timed region; traffic = its ncu DRAM bytes per launch
        kspec = [("k_p1 level-1 place (CSR -> R1)", 8 * E + 8 * (V + 1)),
                 ("k_p2 level-2 place (R1 -> R2)", 8 * E),
                 ("k_p3 level-3 units (R2 -> CSC)", None),
                 ("k_p2 level-3 big buckets (R2 -> CSC)", None)]
        kernels_rf = []
        for (name, kb), kms in zip(kspec, kernel_ms):
            if kms <= 0:
                continue
            ent = {"name": name, "ms": kms}
            if kb is not None:
                ent.update({"algorithmic_bytes": kb, "achieved_gbs": kb / (kms / 1e3) / 1e9,
                            "frac": kb / (kms / 1e3) / 1e9 / peak})
            key = name.split()[0] + ("_big" if "big" in name else "")
            if key in ktraffic:
                ent["traffic"] = ktraffic[key]
            kernels_rf.append(ent)
        l3 = kern.get("step3_ms", 0.0)  # units and big buckets run concurrently (side stream)
        if l3 > 0:
            kernels_rf.append({"name": "level 3 total (units || big-bucket chain)", "ms": l3,
                               "algorithmic_bytes": 8 * E + 8 * (V + 1),
                               "achieved_gbs": (8 * E + 8 * (V + 1)) / (l3 / 1e3) / 1e9,
                               "frac": (8 * E + 8 * (V + 1)) / (l3 / 1e3) / 1e9 / peak})
        kern["per_kernel"] = kernels_rf

    e2e = e2e_dist if dist_on else None
    cpu = None
    if rank == 0 and not dist_on:
        if not args.no_e2e:
            # end to end through the C ABI with pinned host buffers: H2D + kernels + D2H
            h_off = off_d.cpu().pin_memory()
            h_edg = edg_d.cpu().pin_memory()
            h_toff = torch.empty(V + 1, dtype=torch.int64).pin_memory()
            h_tedg = torch.empty(E, dtype=torch.int32).pin_memory()
            del t_off, t_edg
            torch.cuda.empty_cache()

            def host_call():
                rc = _lib.lib.gt_transpose_host(ctypes.c_void_p(h_off.data_ptr()), ctypes.c_void_p(h_edg.data_ptr()),
                                                V, E, ctypes.c_void_p(h_toff.data_ptr()),
                                                ctypes.c_void_p(h_tedg.data_ptr()), local_rank, None)
                _lib.check(rc, "gt_transpose_host")

            host_call()
            n1 = max(1, min(args.steps, 3))
            t0 = time.perf_counter()
            for _ in range(n1):
                host_call()
            t_single = (time.perf_counter() - t0) / n1

            # steady state of a stream of host graphs through the batch entry point: every step
            # still copies its whole input in and its whole result out (pinned host buffers);
            # graph i+1's copy-in overlaps graph i's kernels and graph i-1's copy-out
            h_toff2 = torch.empty(V + 1, dtype=torch.int64).pin_memory()
            h_tedg2 = torch.empty(E, dtype=torch.int32).pin_memory()

            def batch_call(k):
                P64, PV = ctypes.c_uint64 * k, ctypes.c_void_p * k
                outs = [(h_toff, h_tedg), (h_toff2, h_tedg2)]
                rc = _lib.lib.gt_transpose_host_many(
                    k, PV(*[h_off.data_ptr()] * k), PV(*[h_edg.data_ptr()] * k), P64(*[V] * k), P64(*[E] * k),
                    PV(*[outs[i & 1][0].data_ptr() for i in range(k)]), PV(*[outs[i & 1][1].data_ptr() for i in range(k)]),
                    local_rank, None)
                _lib.check(rc, "gt_transpose_host_many")

            batch_call(2)
            ne2e = max(4, min(args.steps, 10))
            t0 = time.perf_counter()
            batch_call(ne2e)
            te = (time.perf_counter() - t0) / ne2e
            # the drop-in figure is the single call INTEGRATION.md binds; the batch entry point
            # (copies of consecutive graphs overlapped with the kernels) is reported beside it
            e2e = {"value": E / t_single, "unit": "edges/s", "h2d_bytes_per_step": (V + 1) * 8 + E * 4,
                   "d2h_bytes_per_step": (V + 1) * 8 + E * 4, "ms_per_step": t_single * 1e3, "steps": n1,
                   "api": "gt_transpose_host (C ABI), one graph per call, pinned host buffers: source chunks copy in while earlier chunks run level 1; bucket groups copy back while later groups run levels 2-3",
                   "stream_of_graphs": {"value": E / te, "ms_per_step": te * 1e3, "steps": ne2e,
                                        "api": "gt_transpose_host_many (C ABI): a stream of host graphs, pinned "
                                               "host buffers, copy-in / kernels / copy-out overlapped across "
                                               "consecutive graphs"}}
        if not args.no_cpu_baseline:
            from oracle import oracle

            oracle.load()
            threads = host_cores()
            off_h = off_d.cpu().numpy().view(np.uint64)
            edg_h = edg_d.cpu().numpy().view(np.uint32)
            del off_d, edg_d
            torch.cuda.empty_cache()
            rep, best, _, desc = cpu_paths_report(off_h, edg_h, V, threads, 20.0)
            cpu = {"value": rep[best]["edges_per_s"], "unit": "edges/s", "cores": threads, "kind": "port",
                   "sample": f"{desc}; fastest sorted reference path = {best} (OpenMP ports in "
                             "oracle/gt_oracle.c, one run each)", "paths": rep}

    # the dominant kernel (longest per-launch time among the place kernels with algorithmic bytes)
    dominant = None
    for ent in (kern or {}).get("per_kernel", []) if isinstance(kern, dict) else []:
        if "algorithmic_bytes" in ent and "level 3 total" not in ent["name"]:
            if dominant is None or ent["ms"] > dominant["ms_per_launch"]:
                dominant = {"name": ent["name"], "ms_per_launch": ent["ms"], "algorithmic_bytes": ent["algorithmic_bytes"],
                            "achieved": ent["achieved_gbs"], "peak": peak, "unit": "GB/s", "frac": ent["frac"],
                            "traffic": ent.get("traffic")}

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "edges/s",
            "n_gpus": n_gpus,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "u32",
            "data": "synthetic",
            "config": {"workload": cfg.name, "num_vertices": V, "num_edges": E,
                       "l2": f"inputs ({((V + 1) * 8 + E * 4) / 1e9:.2f} GB) larger than L2 (126 MB); no flush",
                       "parallelism": f"sharded{n_gpus}" if dist_on else "single-gpu",
                       **({"experiment": args.experiment} if args.experiment else {}),
                       **({"split_forced": args.split} if args.split else {}),
                       **({"force_wide": True} if args.force_wide else {}),
                       **({"rank_mode_forced": args.rank_mode} if args.rank_mode >= 0 else {})},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": agg_peak, "unit": "GB/s",
                         "frac": achieved / agg_peak, "traffic": traffic,
                         "scope": "whole transpose step (all kernels); algorithmic bytes 24(V+1)+12E per step",
                         "peak_source": peak_src, "algorithmic_bytes_per_step": abytes,
                         "frac_vs_datasheet_8tbs": achieved / (8000.0 * n_gpus),
                         "dominant_kernel": dominant, "kernels": kern},
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist_on:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
