"""CLI: python -m paper_2509_24663_b200 {check,bench,quality,gen-fixtures}
  --seed <u64> --config <json> --out <dir> --modes <list> --sizes <list> --precision {f32,f64}
Exit codes: 0 success, 1 tolerance breach, 2 usage / config error."""

from __future__ import annotations

import argparse
import json
import os
import sys


def _cfg(path):
    from .core import AttentionConfig, validate_config
    if path is None:
        return AttentionConfig()
    with open(path) as fh:
        fields = json.load(fh)
    cfg = AttentionConfig(**fields)   # field names mirror AttentionConfig exactly
    validate_config(cfg)
    return cfg


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2509_24663_b200")
    ap.add_argument("command", choices=["check", "bench", "quality", "gen-fixtures"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--config", default=None)
    ap.add_argument("--out", default=".")
    ap.add_argument("--modes", default=None)
    ap.add_argument("--sizes", default=None)
    ap.add_argument("--precision", choices=["f32", "f64"], default="f32")
    ap.add_argument("--perturb", type=float, default=0.0, help=argparse.SUPPRESS)  # test hook
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 2 if e.code else 0
    import numpy as np

    from . import bench_cli as bc
    from .core import ConfigError, atomic_write_bytes
    try:
        cfg = _cfg(args.config)
        sizes = [int(x) for x in args.sizes.split(",") if x] if args.sizes else None
        modes = tuple(args.modes.split(",")) if args.modes else bc.BENCH_MODES
    except (ConfigError, ValueError, TypeError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    os.makedirs(args.out, exist_ok=True)
    prec = np.float64 if args.precision == "f64" else np.float32
    try:
        if args.command == "check":
            rep = bc.run_correctness(args.seed, sizes if sizes is not None else (300, 4096, 8192),
                                     perturb=args.perturb)
            atomic_write_bytes(os.path.join(args.out, "check.json"),
                               json.dumps(rep, indent=2).encode() + b"\n")
            if rep["warning"]:
                print(f"warning: {rep['warning']}", file=sys.stderr)
            return 0 if rep["ok"] else 1
        if args.command == "bench":
            recs = bc.run_bench(cfg, sizes or (4096, 32768, 131072), modes, args.seed)
            bc.write_bench_csv(recs, os.path.join(args.out, "bench.csv"))
            bc.write_bench_json(recs, os.path.join(args.out, "bench.json"))
            return 0
        if args.command == "quality":
            rep = bc.run_selection_quality(cfg, (sizes or [8192])[0], args.seed)
            atomic_write_bytes(os.path.join(args.out, "quality.json"),
                               json.dumps(rep, indent=2).encode() + b"\n")
            return 0 if rep["recall"]["exact"] >= rep["recall"]["random"] else 1
        bc.generate_fixtures(args.out, sizes or (256,), args.seed, cfg, prec)
        return 0
    except (ConfigError, ValueError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
