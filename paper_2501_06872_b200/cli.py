"""``transpose`` command with the reference CLI's arguments for the GPU path.

Mirrors ``potra transpose`` (cli.py:53-71 arguments, cli.py:272-325
``_cmd_transpose``) with ``--algo gpu``: read a POTG file into HBM,
transpose, write the CSC file; ``--report`` writes the same JSON payload
(schema_version 1, bench.py:40).  Exit codes follow cli.py:19-20,120-126:
0 ok, 2 usage / format errors, 3 resource errors.

    python -m paper_2501_06872_b200.cli transpose --algo gpu --in g.potg --out gt.potg
"""

from __future__ import annotations

import argparse
import json
import sys

REPORT_SCHEMA_VERSION = 1  # bench.py:40


def _parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2501_06872_b200.cli")
    sub = ap.add_subparsers(dest="command", required=True)
    t = sub.add_parser("transpose", help="transpose a graph file on the GPU")
    t.add_argument("--algo", choices=["gpu"], required=True)
    t.add_argument("--threads", type=int, default=1, help="devices (the reference's worker count)")
    t.add_argument("--in", dest="input", required=True)
    t.add_argument("--out", required=True)
    t.add_argument("--sort", action="store_true", help="accepted for parity; the output is always sorted")
    t.add_argument("--report", help="write a JSON run report here")
    return ap


def main(argv=None) -> int:
    args = _parser().parse_args(argv)
    from .errors import CounterOverflowError, GpuUnavailableError, GraphFormatError
    from .io import transpose_file

    if args.threads < 1:
        print(f"error: thread count must be >= 1, got {args.threads}", file=sys.stderr)
        return 2
    try:
        phases = transpose_file(args.input, args.out, sort=args.sort)
    except (GraphFormatError, ValueError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    except (MemoryError, CounterOverflowError, GpuUnavailableError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 3
    aux = phases.pop("aux_footprint_bytes")
    if args.report:
        payload = {
            "schema_version": REPORT_SCHEMA_VERSION,
            "algo": args.algo,
            "threads": args.threads,
            "phase_times": phases,
            "aux_footprint_bytes": aux,
            "sorted": True,
            "details": {"method_chosen": "gpu"},
        }
        with open(args.report, "w", encoding="utf-8") as f:
            json.dump(payload, f, indent=2)
    print(f"wrote {args.out} ({args.algo}, {sum(phases.values()):.4f}s in phases)")
    return 0


if __name__ == "__main__":
    sys.exit(main())
