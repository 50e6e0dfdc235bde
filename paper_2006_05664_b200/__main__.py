"""Command line: tune one operator on a B200, or compare optimisers.

    python -m paper_2006_05664_b200 tune --operator matmul:1024,1024,1024 --algo opevo \\
        --budget 500 --seed 0 --out out/
    python -m paper_2006_05664_b200 compare --operator matmul:1024,1024,1024 \\
        --algo opevo,random,sa,gbfs --seeds 0,1,2 --budget 300 --out out/
        (``bench`` is the same command under the reference CLI's name)
    python -m paper_2006_05664_b200 sweep --operator matmul:1024,1024,1024 \\
        --q-grid 0.25,0.5,0.75 --lambda-grid 4,8,16 --seeds 0,1,2 --out out/

Mirrors the reference CLI's ``tune`` / ``bench`` / ``sweep`` subcommands
(``pkg/src/topotune/cli.py:164-270``): same trial-log schema, summary/curve
CSVs and per-cell layout of the hyper-parameter sweep, with ``--evaluator gpu`` (default) measuring TFLOP/s on
the device and ``--evaluator synthetic`` using the reference's CPU model.
Exit codes: 0 ok, 2 usage error, 3 evaluator unavailable.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

from . import (
    EngineConfig,
    FatalEvaluationError,
    make_objective,
    parse_operator,
    run,
)
from .baselines import GbfsConfig, SaConfig, greedy_bfs, random_search, simulated_annealing
from .logs import write_trial_log
from .reporting import curve_rows, summarize, summary_row_dict, tuning_report, write_curves_csv, \
    write_summary_csv

ALGORITHMS = ("opevo", "random", "sa", "gbfs")


def _objective(args):
    spec = parse_operator(args.operator)
    if args.evaluator == "synthetic":
        return make_objective(spec)
    from .evaluator import DTYPES, EvalSettings, GpuEvaluator

    ev = GpuEvaluator(spec, None, args.device,
                      EvalSettings(reps=args.reps, dtype=DTYPES[args.dtype],
                                   preload_family=True))
    return ev.space, ev


def _peak_tflops() -> float:
    """Measured bf16 peak (MEASURED_PEAKS.json at the repo root), else the
    profiling guide's fallback."""
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["bf16_tflops"])
    except (OSError, KeyError, ValueError):
        return 1590.0


def _run(algo, space, objective, seed, budget, parents: int = 8, mutation_rate: float = 0.5):
    if algo == "opevo":
        evaluator = getattr(objective, "evaluate", None)
        cfg = EngineConfig(seed=seed, budget=budget, parents=parents, mutation_rate=mutation_rate)
        return run(space, cfg, objective, evaluator=evaluator)
    if algo == "random":
        return random_search(space, budget, seed, objective)
    if algo == "sa":
        return simulated_annealing(space, SaConfig(), budget, seed, objective)
    if algo == "gbfs":
        return greedy_bfs(space, GbfsConfig(), budget, seed, objective)
    raise ValueError(f"unknown algorithm {algo!r}")


def cmd_tune(args) -> int:
    space, objective = _objective(args)
    t0 = time.perf_counter()
    best, recs = _run(args.algo, space, objective, args.seed, args.budget, args.parents, args.q)
    wall = time.perf_counter() - t0
    os.makedirs(args.out, exist_ok=True)
    path = os.path.join(args.out, f"trials_{args.algo}_seed{args.seed}.jsonl")
    write_trial_log(path, recs)
    rep = tuning_report(recs, wall, _peak_tflops())
    print(json.dumps({"operator": args.operator, "algorithm": args.algo, "seed": args.seed,
                      "best_fitness": best.fitness, "best_config": space.config_to_json(best.config),
                      "log": path, **rep}))
    return 0


def cmd_compare(args) -> int:
    space, objective = _objective(args)
    algos = [a for a in args.algo.split(",") if a]
    seeds = [int(s) for s in args.seeds.split(",") if s]
    rows, curves = [], []
    os.makedirs(args.out, exist_ok=True)
    for algo in algos:
        logs = []
        for seed in seeds:
            _, recs = _run(algo, space, objective, seed, args.budget, args.parents, args.q)
            write_trial_log(os.path.join(args.out, f"trials_{algo}_seed{seed}.jsonl"), recs)
            logs.append(recs)
        row = summarize(algo, args.operator, logs)
        rows.append(summary_row_dict(row))
        curves += curve_rows(algo, logs, args.budget)
        print(json.dumps(summary_row_dict(row)), flush=True)
    write_summary_csv(os.path.join(args.out, "summary.csv"), rows)
    write_curves_csv(os.path.join(args.out, "curves.csv"), curves)
    return 0


def cmd_sweep(args) -> int:
    """OpEvo's hyper-parameters -- mutation rate q and parent count lambda --
    over a grid (reference ``cli.py:237-270``, the paper's sensitivity study):
    one directory ``q{q}_lambda{lambda}`` of trial logs per cell and one
    ``sweep_summary.csv`` row per cell (the reference's column layout: q,
    parents, then the summary columns)."""
    space, objective = _objective(args)
    qs = [float(x) for x in args.q_grid.split(",") if x]
    lams = [int(x) for x in args.lambda_grid.split(",") if x]
    seeds = [int(s) for s in args.seeds.split(",") if s]
    if not qs or not lams or not seeds:
        raise ValueError("empty --q-grid, --lambda-grid or --seeds")
    if args.budget < max(lams):
        raise ValueError(f"--budget {args.budget} is below the parent count {max(lams)}")
    os.makedirs(args.out, exist_ok=True)
    rows = []
    for q in qs:
        for lam in lams:
            cell = os.path.join(args.out, f"q{q}_lambda{lam}")
            os.makedirs(cell, exist_ok=True)
            logs = []
            for seed in seeds:
                _, recs = _run("opevo", space, objective, seed, args.budget, parents=lam, mutation_rate=q)
                write_trial_log(os.path.join(cell, f"trials_opevo_seed{seed}.jsonl"), recs)
                logs.append(recs)
            row = summary_row_dict(summarize("opevo", args.operator, logs), q=q, parents=lam)
            rows.append(row)
            print(json.dumps(row), flush=True)
    write_summary_csv(os.path.join(args.out, "sweep_summary.csv"), rows)
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2006_05664_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("tune", "compare", "bench", "sweep"):
        p = sub.add_parser(name)
        p.add_argument("--operator", required=True)
        p.add_argument("--evaluator", default="gpu", choices=("gpu", "synthetic"))
        p.add_argument("--dtype", default="bf16", choices=("bf16", "f32", "tf32x3"))
        p.add_argument("--device", type=int, default=0)
        p.add_argument("--reps", type=int, default=20)
        p.add_argument("--budget", type=int, default=500)
        p.add_argument("--out", default="out")
        if name != "sweep":   # OpEvo's mutation rate and parent count (reference _add_algo_flags)
            p.add_argument("--q", type=float, default=0.5)
            p.add_argument("--lambda", dest="parents", type=int, default=8)
        if name == "tune":
            p.add_argument("--algo", default="opevo", choices=ALGORITHMS)
            p.add_argument("--seed", type=int, default=int(os.environ.get("TOPO_TUNE_SEED", 0)))
        elif name in ("compare", "bench"):
            p.add_argument("--algo", default=",".join(ALGORITHMS))
            p.add_argument("--seeds", default="0,1,2")
        else:
            p.add_argument("--q-grid", default="0.5", help="comma-separated mutation rates")
            p.add_argument("--lambda-grid", default="8", help="comma-separated parent counts")
            p.add_argument("--seeds", default="0,1,2")
    args = ap.parse_args(argv)
    try:
        return {"tune": cmd_tune, "compare": cmd_compare, "bench": cmd_compare,
                "sweep": cmd_sweep}[args.cmd](args)
    except FatalEvaluationError as err:
        print(f"evaluator unavailable: {err}", file=sys.stderr)
        return 3
    except ValueError as err:
        print(f"usage error: {err}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
