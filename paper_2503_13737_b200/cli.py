"""Command-line front end (reference SPEC.md:531-594, the `cli` module the shipped package declares
at pyproject.toml:20-21 but does not contain): trace generation, runs of one or more policies,
report comparison, calibration.

  python -m paper_2503_13737_b200.cli gen --out trace.jsonl [--requests N --rate R --long-fraction F --seed S]
  python -m paper_2503_13737_b200.cli run --trace trace.jsonl --policy accelgen --policy paged_fcfs
                                          [--profile P] [--executor virtual|cuda] [--horizon H] --out DIR
  python -m paper_2503_13737_b200.cli compare DIR/report_*.json --baseline paged_fcfs
  python -m paper_2503_13737_b200.cli calibrate --profile P --gpu G --out P2   (derive_pivot rule)
  python -m paper_2503_13737_b200.cli calibrate --measure --out P2             (B200 profiler)

Exit codes: 0 success, 1 configuration error, 2 I/O error, 3 internal invariant fault.
--executor virtual advances the clock by iteration_time(S_f) (the reference semantics); cuda runs
the B200 forward (clock = CUDA-event device time of each step).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
from pathlib import Path

from . import cost_model as cm
from . import workload
from .errors import ConfigError, EngineFault, StateError, TraceParseError, ValidationError

EXIT_OK, EXIT_CONFIG, EXIT_IO, EXIT_FAULT = 0, 1, 2, 3
REPORT_METRICS = ("tokens_per_s", "reqs_per_s", "goodput", "slo_attainment", "jct_slo_attainment", "jct_mean",
                  "gpu_util_mean", "kvc_util_mean")


def _log(msg: str) -> None:
    if os.environ.get("SLOSIM_LOG", "info").lower() not in ("quiet", "error"):
        print(msg, file=sys.stderr)


def cmd_gen(args) -> int:
    """JSONL trace + printed summary."""
    prof = cm.load_profile(args.profile) if args.profile else cm.opt_13b_like()
    cfg = workload.TraceConfig(num_requests=args.requests, arrival_rate=args.rate, long_fraction=args.long_fraction,
                               long_len_dist=workload.LengthDist(kind="log_uniform", lo=args.long_lo, hi=args.long_hi),
                               offline_fraction=args.offline_fraction, seed=args.seed, profile=prof)
    trace = workload.generate_trace(cfg)
    workload.save_trace(trace, args.out)
    print(json.dumps(workload.trace_summary(trace)))
    return EXIT_OK


def _run_one(trace, profile, policy: str, executor_kind: str, horizon: float, kv_blocks: int | None):
    from .engine import Engine
    from .policies import PolicyConfig
    pc = PolicyConfig(policy=policy)
    if executor_kind == "virtual":
        eng = Engine(trace, profile, pc, None, clock="virtual", kv_blocks=kv_blocks, horizon_s=horizon)
    else:
        from . import model as M
        from .executor import CudaExecutor
        mcfg = M.opt_13b(max_positions=max(r.prompt_len + r.output_len for r in trace) + 64) \
            if profile.hidden_size == 5120 else M.opt_175b(max_positions=max(r.prompt_len + r.output_len
                                                                             for r in trace) + 64)
        blocks = kv_blocks or max(1, profile.kvc_capacity_tokens // 32)
        ex = CudaExecutor(mcfg, blocks, max_tokens=max(profile.pivot_forward_size, 16384), max_seqs=2048)
        try:
            return Engine(trace, profile, pc, ex, clock="device", kv_blocks=blocks, horizon_s=horizon).run()
        finally:
            ex.close()  # weights + a KV pool sized to the profile: give the HBM back before the next policy
    return eng.run()


def cmd_run(args) -> int:
    """one MetricsReport JSON + one CSV row per policy."""
    from .engine import CSV_COLUMNS
    if not args.policy:
        raise ConfigError("at least one --policy")
    if args.trace:
        trace = workload.load_trace(args.trace)
    else:
        prof = cm.load_profile(args.profile) if args.profile else cm.opt_13b_like()
        trace = workload.generate_trace(workload.TraceConfig(num_requests=args.requests, arrival_rate=args.rate,
                                                             seed=args.seed, profile=prof))
    profile = cm.load_profile(args.profile) if args.profile else cm.opt_13b_like()
    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    rows = [",".join(CSV_COLUMNS)]
    trace_id = f"{len(trace)}:{sum(r.prompt_len for r in trace)}:{sum(r.output_len for r in trace)}"
    for pol in args.policy:
        rep = _run_one(trace, profile, pol, args.executor, args.horizon, args.kv_blocks)
        d = rep.to_dict()
        d["trace_id"] = trace_id
        (out / f"report_{pol}.json").write_text(json.dumps(d, indent=1))
        rows.append(rep.csv_row())
        _log(f"{pol}: tokens/s {rep.tokens_per_s:.1f} SLO attainment {rep.slo_attainment:.4f}")
    (out / "report.csv").write_text("\n".join(rows) + "\n")
    print("\n".join(rows))
    return EXIT_OK


def cmd_compare(args) -> int:
    """per-metric ratios against a named baseline policy (+ JSON)."""
    reps = [json.loads(Path(p).read_text()) for p in args.reports]
    if len(reps) < 2:
        raise ConfigError("compare needs at least two reports")
    if len({r.get("trace_id") for r in reps}) != 1:
        raise ConfigError("reports come from different traces")
    by = {r["policy"]: r for r in reps}
    if args.baseline not in by:
        raise ConfigError(f"baseline policy {args.baseline!r} not among {sorted(by)}")
    base = by[args.baseline]
    table = {}
    for pol, r in by.items():
        if pol == args.baseline:
            continue
        table[pol] = {m: (r[m] / base[m] if base[m] not in (0, 0.0) else math.inf if r[m] else 1.0)
                      for m in REPORT_METRICS}
    print(json.dumps({"baseline": args.baseline, "ratios": table}, indent=1))
    return EXIT_OK


def cmd_calibrate(args) -> int:
    """complete a profile.  --measure runs the B200 profiler (the sweep the paper
    describes); otherwise S_pf / T_pf come from derive_pivot / derive_pivot_time (reference rule)."""
    if args.measure:
        from . import profiler
        sys.argv = ["profiler", "--out", args.out] + (["--tp", str(args.tp)] if args.tp else [])
        profiler.main()
        return EXIT_OK
    if not args.profile:
        raise ConfigError("calibrate needs --profile (or --measure)")
    raw = json.loads(Path(args.profile).read_text())
    missing = [k for k in ("hidden_size", "num_layers") if k not in raw]
    if missing:
        raise ConfigError(f"profile lacks {missing}")
    if "pivot_forward_size" in raw and "pivot_time_s" in raw:
        prof = cm.load_profile(args.profile)  # complete: idempotent
    else:
        if not args.gpu:
            raise ConfigError("missing keys ['pivot_forward_size', 'pivot_time_s'] and no --gpu profile to derive them")
        gpu = cm.load_gpu_profile(args.gpu)
        s_pf = raw.get("pivot_forward_size") or cm.derive_pivot(raw["hidden_size"], raw["num_layers"], gpu)
        t_pf = raw.get("pivot_time_s") or cm.derive_pivot_time(s_pf, raw["hidden_size"], raw["num_layers"], gpu)
        prof = cm.ModelProfile(**{**raw, "pivot_forward_size": int(s_pf), "pivot_time_s": float(t_pf)})
    cm.save_profile(prof, args.out)
    print(json.dumps(prof.__dict__))
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="accelgen-b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    g = sub.add_parser("gen")
    g.add_argument("--out", required=True)
    g.add_argument("--requests", type=int, default=1000)
    g.add_argument("--rate", type=float, default=8.0)
    g.add_argument("--long-fraction", type=float, default=0.35)
    g.add_argument("--offline-fraction", type=float, default=0.0)
    g.add_argument("--long-lo", type=int, default=4096)
    g.add_argument("--long-hi", type=int, default=100000)
    g.add_argument("--seed", type=int, default=0)
    g.add_argument("--profile", default=None)
    r = sub.add_parser("run")
    r.add_argument("--trace", default=None)
    r.add_argument("--requests", type=int, default=200)
    r.add_argument("--rate", type=float, default=8.0)
    r.add_argument("--seed", type=int, default=0)
    r.add_argument("--policy", action="append", default=[])
    r.add_argument("--profile", default=None)
    r.add_argument("--executor", choices=("virtual", "cuda"), default="virtual")
    r.add_argument("--horizon", type=float, default=math.inf)
    r.add_argument("--kv-blocks", type=int, default=None)
    r.add_argument("--out", required=True)
    c = sub.add_parser("compare")
    c.add_argument("reports", nargs="+")
    c.add_argument("--baseline", required=True)
    k = sub.add_parser("calibrate")
    k.add_argument("--profile", default=None)
    k.add_argument("--gpu", default=None)
    k.add_argument("--measure", action="store_true")
    k.add_argument("--tp", type=int, default=None)
    k.add_argument("--out", required=True)
    return ap


BUILTIN_PROFILES = ("opt-13b", "opt-175b")


def main(argv=None) -> int:
    try:
        args = build_parser().parse_args(argv)
    except SystemExit as e:  # argparse usage errors are configuration errors
        return EXIT_CONFIG if e.code not in (0, None) else EXIT_OK
    for attr in ("profile", "gpu", "trace"):  # missing input files are I/O errors
        path = getattr(args, attr, None)
        if path and path not in BUILTIN_PROFILES and not Path(path).exists():
            print(f"I/O error: {attr} file not found: {path}", file=sys.stderr)
            return EXIT_IO
    fn = {"gen": cmd_gen, "run": cmd_run, "compare": cmd_compare, "calibrate": cmd_calibrate}[args.cmd]
    try:
        return fn(args)
    except (ConfigError, ValidationError) as e:
        print(f"configuration error: {e}", file=sys.stderr)
        return EXIT_CONFIG
    except (OSError, TraceParseError) as e:
        print(f"I/O error: {e}", file=sys.stderr)
        return EXIT_IO
    except (EngineFault, StateError) as e:
        print(f"internal invariant fault: {e}", file=sys.stderr)
        return EXIT_FAULT


if __name__ == "__main__":
    sys.exit(main())
