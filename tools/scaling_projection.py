"""Project 1/2/4/8-GPU trial throughput from one GPU (a measurement aid for a
box with one GPU; the real multi-GPU run is ``torchrun ... bench.py --gpus N``).

Under ``scheduler.ShardedEvaluator`` every rank runs the same engine replica
(the native proposal core) and evaluates ask indices i = rank (mod N); a
generation ends when the slowest rank has its shard and one small all-reduce
has gathered the rows.  Here:

1. a reference run measures every trial of the search on this GPU and
   records its fitness;
2. for each N, the same trajectory is replayed (recorded fitness told, so the
   asks are identical); every simulated rank has its own evaluator -- its own
   operand, verification record and straggler-rule state, as a real rank
   has -- sharing this GPU's context and loaded kernels, and generation by
   generation each rank's shard is measured on the GPU in turn, together
   with the host ask/tell of that generation;
3. the projected generation time is the max over ranks plus a fixed
   all-reduce latency (``--allreduce-us``: the host gloo exchange of an
   8 x 11 fp64 table, measured ~30-60 us on loopback).

Usage: python tools/scaling_projection.py [op] [generations]
"""
import argparse
import json
import os
import sys
import time


sys.path.insert(0, ".")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("op", nargs="?", default="matmul:1024,1024,1024")
    ap.add_argument("generations", nargs="?", type=int, default=40)
    ap.add_argument("--allreduce-us", type=float, default=30.0)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--timing", default="stream", choices=("stream", "graph"),
                    help="fitness launches: gated stream (bench default) or one CUDA graph per trial")
    args = ap.parse_args()

    from paper_2006_05664_b200 import EngineConfig, parse_operator
    from paper_2006_05664_b200.evaluator import EvalSettings, GpuEvaluator
    from paper_2006_05664_b200.mapping import gpu_operator_space
    from paper_2006_05664_b200.native import NativeOpEvo
    from paper_2006_05664_b200.scheduler import shard_indices

    spec = parse_operator(args.op)
    space = gpu_operator_space(spec)
    mode = 2 if args.timing == "stream" else 0
    ev = GpuEvaluator(spec, space, 0, EvalSettings(preload_family=True, flush_l2=mode))
    warm = 3
    budget = 8 * (args.generations + warm)

    # 1. reference run: fitness of every asked configuration
    fitness = {}
    order = []                      # fitness in trial order (identical at every N)
    eng = NativeOpEvo(space, EngineConfig(seed=args.seed, budget=budget))
    while True:
        a = eng.ask()
        if not a.configs:
            break
        fits = ev.evaluate(a.configs)
        for c, f in zip(a.configs, fits):
            fitness[c] = f
            order.append(f)
        eng.tell(list(zip(a.configs, fits)))
    # the first trial whose running best reaches 95 % of the final best
    # (reference reporting.py:33-41); its generation index
    final_best = max(order) if order else 0.0
    run_best, t95 = 0.0, len(order)
    for i, f in enumerate(order):
        run_best = max(run_best, f)
        if run_best >= 0.95 * final_best:
            t95 = i + 1
            break
    gen_of_t95 = (t95 - 1) // 8

    out = {"op": args.op, "generations": args.generations, "allreduce_us": args.allreduce_us,
           "timing": args.timing,
           "seed": args.seed, "per_n": {}}
    for n in (1, 2, 4, 8):
        ranks = [GpuEvaluator(spec, space, 0, EvalSettings(flush_l2=mode), dev=ev.dev) for _ in range(n)]
        eng = NativeOpEvo(space, EngineConfig(seed=args.seed, budget=budget))
        gen_ms, rank_ms, all_gen_ms = [], [], []
        trials = 0
        g = 0
        while True:
            ev.dev.flush_l2()
            t0 = time.perf_counter()
            a = eng.ask()
            t_ask = time.perf_counter() - t0
            if not a.configs:
                break
            rank_s = []
            for r in range(n):
                idx = shard_indices(len(a.configs), n, r)
                t1 = time.perf_counter()
                if idx:
                    ranks[r].evaluate([a.configs[i] for i in idx])
                rank_s.append(time.perf_counter() - t1)
            t2 = time.perf_counter()
            eng.tell([(c, fitness[c]) for c in a.configs])   # recorded: identical trajectory
            t_tell = time.perf_counter() - t2
            all_gen_ms.append(1e3 * (t_ask + max(rank_s) + t_tell) + (args.allreduce_us / 1e3 if n > 1 else 0))
            if g >= warm:
                gen_ms.append(all_gen_ms[-1])
                rank_ms.append(1e3 * max(rank_s))
                trials += len(a.configs)
            g += 1
        for r in ranks:
            r.close()
        tot = sum(gen_ms)
        out["per_n"][n] = {"trials": trials, "ms_per_generation": tot / max(1, len(gen_ms)),
                           "ms_slowest_rank": sum(rank_ms) / max(1, len(rank_ms)),
                           "trials_per_s": trials / (tot / 1e3) if tot else 0.0,
                           # identical trajectory at every N: the same best and the same
                           # trial reaches 95 % of it; only the wall clock differs
                           "best_tflops": final_best, "trials_to_95pct": t95,
                           "wallclock_to_95pct_ms": sum(all_gen_ms[:gen_of_t95 + 1])}
        print(f"N={n}: {out['per_n'][n]['ms_per_generation']:.3f} ms/generation "
              f"(slowest rank {out['per_n'][n]['ms_slowest_rank']:.3f}), "
              f"{out['per_n'][n]['trials_per_s']:.0f} trials/s; best {final_best:.1f} TFLOP/s, "
              f"95 % of it at trial {t95} after {out['per_n'][n]['wallclock_to_95pct_ms']:.2f} ms",
              flush=True)
    base = out["per_n"][1]["trials_per_s"]
    for n in (2, 4, 8):
        out["per_n"][n]["speedup_vs_1"] = out["per_n"][n]["trials_per_s"] / base if base else 0.0
    print(json.dumps(out))
    ev.close()


if __name__ == "__main__":
    main()
