#!/usr/bin/env python
"""Benchmark: OpEvo tuning of an sm_100a kernel family on B200.

A *step* is one OpEvo generation of the reference loop (ask rho=8 configs ->
evaluate them on the GPUs -> tell), i.e. the hot path of ``run``
(reference ``pkg/src/topotune/engine.py:293-310``) with the trial evaluator
replaced by compile + verify + CUDA-event timing of a tcgen05/TMA kernel.

``value`` = trials/s over the K timed generations (whole job, all ranks);
the best-found TFLOP/s, its fraction of the measured tensor-core peak,
trials-to-95 % and wall-clock-to-95 % of the best ride along.  Default
workload: BASELINE configs[1], MatMul 1024x1024x1024 bf16.

N > 1: launched by torchrun, one process per GPU; every rank runs an
identical engine replica and evaluates the ask indices i = rank (mod N); one
all_reduce of the result rows per generation (scheduler.ShardedEvaluator).

``--impl reference``: the reference's own CPU path (OpEvo + its synthetic CPU
evaluator): the unmodified reference package installed into baseline/_ref
(tools/install_reference.sh), or its restatement oracle/opevo_port.py when
that install is absent; rank 0 only, on the host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

RHO = 8
DEFAULT_OP = "matmul:1024,1024,1024"
METRIC = "best-found TFLOP/s (% of tensor peak) vs trials; trials/sec at 1/2/4/8 B200"
# CUDA-core fp32 FMA peak: 148 SMs x 128 lanes x 2 flop x 1.965 GHz (nominal
# clock; no measured figure exists for this pipe)
FP32_PEAK = 148 * 128 * 2 * 1.965e9 / 1e12


def peaks() -> dict:
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return {"tflops": p["bf16_tflops"], "tflops_sustained": p.get("bf16_tflops_sustained"),
                "hbm_gbs": p["hbm_gbs"], "source": "measured"}
    except (OSError, KeyError, ValueError):
        return {"tflops": 1590.0, "tflops_sustained": 1400.0, "hbm_gbs": 6650.0,
                "source": "fallback"}


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region.

    In-process NVML (nvidia-ml-py) polled every 20 ms: a handful of fields
    per sample.  A looping ``nvidia-smi`` (the fallback) queries many fields
    per sample and was seen to stall concurrent driver calls (module loads,
    graph instantiation) by tens of milliseconds, which shows up as noise in
    the trials/s of this short timed region."""

    # NVML clocks-event reason bits
    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}
    FIELDS = ("index,clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int, period_s: float = 0.02):
        self.gpu = gpu
        self.period = period_s
        self.proc = None
        self.nvml = None
        self.rows: list[tuple] = []      # (sm_mhz, max_mhz, util, reason_bits)
        self.lines: list[str] = []       # nvidia-smi fallback
        self.stop = threading.Event()

    def __enter__(self):
        if os.environ.get("OPEVO_NO_CLOCKS") == "1":      # diagnostics only
            return self
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.sample()
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception:   # noqa: BLE001 - NVML unavailable: nvidia-smi
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def sample(self):
        n = self.nvml
        try:
            sm = n.nvmlDeviceGetClockInfo(self.h, n.NVML_CLOCK_SM)
            util = n.nvmlDeviceGetUtilizationRates(self.h).gpu
            try:
                bits = n.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except AttributeError:
                bits = n.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
            self.rows.append((float(sm), float(self.max_mhz), float(util), int(bits)))
        except Exception:   # noqa: BLE001
            pass

    def _poll(self):
        while not self.stop.wait(self.period):
            self.sample()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.nvml is not None:
            self.stop.set()
            self.t.join(timeout=2)
            self.sample()
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self) -> dict:
        if self.rows:
            sm = [r[0] for r in self.rows]
            loaded = [r[0] for r in self.rows if r[2] > 0] or sm
            reasons = sorted({name for r in self.rows for name, bit in self.REASONS.items() if r[3] & bit})
            return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": self.rows[0][1],
                    "reasons": reasons, "samples": len(self.rows), "source": "nvml"}
        rows = []
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        util = [float(r[3]) for r in rows if r[3].replace(".", "").isdigit()]
        loaded = [s for s, u in zip(sm, util) if u > 0] or sm
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v == "Active"})
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows), "source": "nvidia-smi"}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


REF_DIR = os.path.join(REPO, "baseline", "_ref")


def _stock_reference():
    """The unmodified reference package (topotune 0.1.0) installed into
    baseline/_ref by tools/install_reference.sh, or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "topotune")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import topotune
        from topotune import benchmarks, engine
    except ImportError:
        return None
    if not os.path.abspath(topotune.__file__).startswith(REF_DIR):
        return None
    return engine, benchmarks


def cpu_reference_arm(op: str, budget: int, seed: int, max_s: float = 10.0) -> dict:
    """The reference's CPU search + synthetic evaluator, timed on this host:
    the stock ``topotune.run(space, EngineConfig(seed, budget), objective)``
    with ``make_objective`` (reference engine.py:293-310, benchmarks.py:294-302)
    from baseline/_ref, or -- when that install is absent -- its restatement
    oracle/opevo_port.py.  One thread: a search is one serial ask/tell chain,
    and the reference's ``concurrency`` knob (a thread pool over the objective
    calls) measured slower than serial for its microsecond objective
    (6.5 k vs 3.9 k trials/s with 8 threads on the build host).  Each run is
    one search of ``budget`` trials (our arm's search budget)."""
    stock = _stock_reference()
    if stock is not None:
        engine, benchmarks = stock
        space, objective = benchmarks.make_objective(benchmarks.parse_operator(op))

        def one(s):
            _, recs = engine.run(space, engine.EngineConfig(seed=s, budget=budget), objective)
            return len(recs)
        kind, what = "reference", ("the unmodified reference (stock topotune 0.1.0 from baseline/_ref): "
                                   "topotune.engine.run with benchmarks.make_objective")
    else:
        from oracle import opevo_port

        def one(s):
            return len(opevo_port.opevo_run(op, seed=s, budget=budget)[1])
        kind, what = "port", "the reference's loop restated in oracle/opevo_port.py (baseline/_ref absent)"
    reps, total_s, trials = 0, 0.0, 0
    t_end = time.perf_counter() + max_s
    while True:
        t0 = time.perf_counter()
        trials += one(seed + reps)
        total_s += time.perf_counter() - t0
        reps += 1
        if time.perf_counter() > t_end or reps >= 2000:
            break
    return {"value": trials / total_s, "unit": "trials/s", "cores": 1, "kind": kind,
            "stock": stock is not None,
            "sample": f"{reps} OpEvo runs x {budget} trials of {op} with the reference's synthetic "
                      f"CPU evaluator: {what}; 1 thread, {total_s:.1f} s of CPU work",
            "cpu": _cpu_model(), "host_cpus": os.cpu_count()}


_CPU_OP_SCRIPT = r"""
import json, os, sys, time
import torch
kind, dims, dtype, reps = sys.argv[1], [int(x) for x in sys.argv[2].split(",")], sys.argv[3], int(sys.argv[4])
threads = os.cpu_count() or 1
torch.set_num_threads(threads)
tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
g = torch.Generator().manual_seed(1234)
r = lambda *s: torch.rand(*s, generator=g).to(tdt)
if kind == "matmul":
    n, m, k = dims; a, b = r(n, k), r(m, k); fn = lambda: torch.matmul(a, b.t())
elif kind == "batchmatmul":
    bb, n, m, k = dims; a, b = r(bb, n, k), r(bb, m, k); fn = lambda: torch.bmm(a, b.transpose(1, 2))
else:
    n, c, h, w, co, kh, kw, st, pd = dims
    x, f = r(n, c, h, w), r(co, c, kh, kw)
    fn = lambda: torch.nn.functional.conv2d(x, f, stride=st, padding=pd)
fn()
best, t_end = float("inf"), time.perf_counter() + 15.0
for _ in range(reps):
    t0 = time.perf_counter(); fn(); best = min(best, time.perf_counter() - t0)
    if time.perf_counter() > t_end:
        break
print(json.dumps({"best_s": best, "threads": threads}))
"""


def cpu_operator_throughput(op: str, dtype: str = "bf16", reps: int = 30) -> dict | None:
    """SURVEY.md §8d CPU baseline (2): the operator itself on this host's
    cores (torch.matmul / bmm / conv2d with every thread, in a separate
    process), best of `reps`.  A reported baseline for best_tflops, not a
    target."""
    from paper_2006_05664_b200 import parse_operator

    spec = parse_operator(op)
    kind, dims = op.split(":")
    # Best of three processes: on the build container torch's CPU bf16 GEMM
    # ran either ~2.4 or ~0.065 TFLOP/s per process at random (the oneDNN
    # AMX path is picked up or not), so one process can understate the host.
    runs = []
    for _ in range(3):
        try:
            out = subprocess.run([sys.executable, "-c", _CPU_OP_SCRIPT, kind, dims, dtype, str(reps)],
                                 capture_output=True, text=True, timeout=300, check=True)
            runs.append(json.loads(out.stdout.strip().splitlines()[-1]))
        except (subprocess.SubprocessError, ValueError, IndexError):
            continue
    if not runs:
        return None
    r = min(runs, key=lambda x: x["best_s"])
    fn = {"matmul": "matmul", "batchmatmul": "bmm", "conv2d": "conv2d"}[kind]
    return {"value": spec.flops() / r["best_s"] / 1e12, "unit": "TFLOP/s", "cores": r["threads"],
            "impl": f"torch.{fn} {'bf16' if dtype == 'bf16' else 'fp32'} on the host CPU",
            "sample": f"best of {reps} calls of {op}, best of {len(runs)} processes",
            "per_process_tflops": [spec.flops() / x["best_s"] / 1e12 for x in runs]}


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args) -> None:
    world, rank, _ = dist_env()
    if rank != 0:
        return
    budget = max(args.budget, RHO * (args.steps + args.warmup))
    cb = cpu_reference_arm(args.op, budget, args.seed)
    cb["operator"] = cpu_operator_throughput(args.op)
    ms = 1e3 * RHO / cb["value"]
    line = {"metric": METRIC, "value": cb["value"], "unit": "trials/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": f"OpEvo search, {args.op}, reference synthetic CPU evaluator",
                       "operator": args.op, "rho": RHO, "seed": args.seed, "search_budget": budget},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "trials/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "note": "the reference's evaluator is a synthetic cost model (no device meaning, "
                    "SPEC.md:13); its fitness is not TFLOP/s"}
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--op", default=DEFAULT_OP)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--reps", type=int, default=20, help="timed launches per trial")
    ap.add_argument("--budget", type=int, default=500,
                    help="trials of the whole search (the north star's 500); the generations after "
                         "the timed ones complete it untimed")
    ap.add_argument("--loser-ratio", type=float, default=1.2,
                    help="straggler rule: candidates slower than this x the fastest verified one "
                         "are timed with 5 launches (0: off)")
    ap.add_argument("--l2", default="auto", choices=("auto", "warm", "cold"),
                    help="fitness launches with a warm L2, or each after an L2 flush (cold); auto: "
                         "cold for bf16 operators below the ridge (HBM-bound: BMM1), warm otherwise")
    ap.add_argument("--timing", default="stream", choices=("graph", "stream"),
                    help="fitness launches: stream launches released together by a device gate "
                         "(default) or one CUDA graph")
    ap.add_argument("--dtype", default="bf16", choices=("bf16", "f32", "tf32x3"),
                    help="f32: the SIMT family on the reference space (cfg1); tf32x3: fp32 "
                         "operands on the tensor cores (three kind::tf32 MMAs per K step)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-preload", action="store_true",
                    help="do not load the cached kernel family into the context before timing")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-cold", action="store_true", help="skip the cold-kernel-cache sub-record")
    ap.add_argument("--python-ask", action="store_true",
                    help="propose with the Python engine instead of the native core (same proposals)")
    ap.add_argument("--log", default="")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    args.warmup = max(args.warmup, 3)

    world, rank, local = dist_env()
    import torch
    import torch.distributed as dist

    from paper_2006_05664_b200 import EngineConfig, OpEvo, parse_operator
    from paper_2006_05664_b200.evaluator import DTYPES, EvalSettings, GpuEvaluator
    from paper_2006_05664_b200.logs import TrialRecorder
    from paper_2006_05664_b200.mapping import config_to_knobs, gpu_operator_space
    from paper_2006_05664_b200.reporting import trials_to_fraction, wallclock_to_fraction
    from paper_2006_05664_b200.scheduler import ShardedEvaluator

    # OPEVO_DIST_BACKEND=gloo (test mode): ranks may share GPUs and the
    # per-generation exchange goes through host memory; default NCCL
    backend = os.environ.get("OPEVO_DIST_BACKEND", "nccl")
    if backend == "gloo":
        local %= max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    # the per-generation exchange, the barriers and the max over ranks go
    # through shared memory (ShmExchange: ~10-25 us at 2-8 ranks, where a
    # gloo all-reduce of the same table took 1.4-29 ms); a gloo group only
    # sets it up.  No CUDA context is involved, so a rank whose context a
    # faulting candidate poisoned still takes part.
    exch = (dist.new_group(backend="gloo") if backend == "nccl" else None) if world > 1 else None
    from paper_2006_05664_b200 import capi
    from paper_2006_05664_b200.scheduler import ProcessEvaluator, ShmExchange

    xchg = ShmExchange.create(rank, world, group=exch) if world > 1 else None

    spec = parse_operator(args.op)
    space = gpu_operator_space(spec, args.dtype)
    if args.l2 == "auto":
        # tune in the regime the operator's roofline describes: an HBM-bound
        # operator's fitness is its launch with the operands coming from HBM
        pk0 = peaks()
        below = (args.dtype == "bf16"
                 and spec.flops() / algo_bytes(spec, 2) < pk0["tflops"] * 1e3 / pk0["hbm_gbs"])
        args.l2 = "cold" if below else "warm"
    settings = EvalSettings(reps=args.reps, preload_family=not args.no_preload, warm_family=not args.no_preload,
                            flush_l2=1 if args.l2 == "cold" else (2 if args.timing == "stream" else 0),
                            dtype=DTYPES[args.dtype], loser_ratio=args.loser_ratio)
    local_ev = GpuEvaluator(spec, space, local, settings)
    if world > 1:
        evaluator = ShardedEvaluator(local_ev, rank, world, group=exch, exchange=xchg,
                                     respawn=lambda: ProcessEvaluator(spec, space, local, settings))
    else:
        evaluator = local_ev.evaluate

    def poisoned() -> bool:
        return bool(getattr(evaluator, "poisoned", False))

    def flush():
        # enqueued ahead of the step's kernels on the library's stream; the
        # host goes on with the step's ask meanwhile
        if world > 1:
            evaluator.flush_l2()        # the worker process's after a fault
        else:
            local_ev.dev.flush_l2(wait=False)

    def barrier():
        if not poisoned():
            torch.cuda.synchronize()
        if world > 1:
            xchg.barrier()

    def max_over_ranks(x: float) -> float:
        return xchg.max(x) if world > 1 else x

    def launches_of(extras) -> int:
        # tuned-kernel launches reported by the C ABI, plus one compare
        # kernel per trial that ran its check (not for re-timed instances
        # verified earlier on the same operands)
        return sum(int(e.get("launches", 0)) + (1 if e.get("status") in ("ok", "verify_failed")
                                                and not e.get("verify_cached") else 0) for e in extras)

    from paper_2006_05664_b200.native import NativeOpEvo

    def new_search(budget: int):
        # the C++ proposal core (csrc/search.cpp): the reference's proposals,
        # bit for bit, in microseconds (tests/test_native_search.py)
        engine_cls = OpEvo if args.python_ask else NativeOpEvo
        return (engine_cls(space, EngineConfig(seed=args.seed, budget=budget, parents=RHO,
                                               offspring=RHO)),
                TrialRecorder(space))

    history: list[tuple[list, list]] = []      # (asked, told) of every generation of the search

    def generation(eng, rec, upload=None, tally=None, replay=None) -> int:
        """One generation: ask -> evaluate -> tell.  ``replay`` (the
        e2e leg): the recorded (asked, told) of the same generation of the
        search -- the engine is told the recorded fitness, so a fresh engine
        with the same seed asks exactly the same configurations again, and
        they are measured again from scratch."""
        if upload is not None:
            upload()
        asked = eng.ask()
        if not asked.configs:
            return 0
        fits = evaluator(asked.configs)
        if replay is not None:
            if asked.configs != replay[0]:
                raise RuntimeError("e2e replay diverged from the recorded search")
            fits = replay[1]
        else:
            history.append((list(asked.configs), list(fits)))
        eng.tell(list(zip(asked.configs, fits)))
        owner = getattr(evaluator, "__self__", evaluator)
        extras = owner.last_extras
        for c, f, e in zip(asked.configs, fits, extras):
            rec.record(c, f, e)
        if tally is not None:
            tally["launches"] += launches_of(extras)
            tally["valid"] += sum(e.get("status") == "ok" for e in extras)
            tally["verified"] += sum(e.get("status") in ("ok", "verify_failed")
                                     and not e.get("verify_cached") for e in extras)
            tally["instances"].update(tuple(e["knobs"]) for e in extras if e.get("knobs"))
        return len(asked.configs)

    budget = max(args.budget, RHO * (args.steps + args.warmup))
    engine, recorder = new_search(budget)
    for _ in range(args.warmup):
        generation(engine, recorder)

    # ---------------- timed region: K generations, device-timed, max over ranks
    # (the Python garbage collector is paused inside it: a collection pass is
    # host jitter of a few ms against a ~70 ms region)
    import gc

    gc.collect()
    gc.disable()
    barrier()
    trials = 0
    tally = {"launches": 0, "valid": 0, "verified": 0, "instances": set()}
    e0 = e1 = None
    if not poisoned():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        if e0 is not None:
            e0.record()
        t_wall0 = time.perf_counter()
        gen_diag = [] if os.environ.get("OPEVO_BENCH_GEN_TIMES") == "1" else None
        flush_ms = []
        for _ in range(args.steps):
            tf = time.perf_counter()
            flush()                     # every step starts with a cold L2
            tg = time.perf_counter()
            trials += generation(engine, recorder, tally=tally)
            if gen_diag is not None:    # diagnostics: host time per generation + its trials
                owner = getattr(evaluator, "__self__", evaluator)
                gen_diag.append((1e3 * (time.perf_counter() - tg), list(owner.last_extras)))
                flush_ms.append(1e3 * (tg - tf))
        t_loop = time.perf_counter()
        barrier()
        wall = time.perf_counter() - t_wall0
        if gen_diag is not None:
            print(f"[timed region] loop {1e3 * (t_loop - t_wall0):.1f} ms, final barrier "
                  f"{1e3 * (time.perf_counter() - t_loop):.1f} ms", file=sys.stderr)
        timing = "cuda events (max over ranks)"
        try:
            if poisoned() or e0 is None:
                raise RuntimeError("context poisoned")
            e1.record()
            torch.cuda.synchronize()
            local_sec = e0.elapsed_time(e1) / 1e3
        except RuntimeError:
            # a faulting candidate poisoned this rank's CUDA context mid-run
            # (its evaluation moved to a worker process): events are gone
            local_sec = wall
            timing = f"host wall clock on rank {rank} (CUDA context poisoned by a faulting candidate)"
    gc.enable()
    if gen_diag:
        slow = sorted(range(len(gen_diag)), key=lambda i: -gen_diag[i][0])[:3]
        med = statistics.median(t for t, _ in gen_diag)
        print("[gen ms] " + " ".join(f"{t:.2f}" for t, _ in gen_diag), file=sys.stderr)
        print(f"[flush] median {statistics.median(flush_ms):.3f} ms, max {max(flush_ms):.3f} ms, "
              f"total {sum(flush_ms):.1f} ms; generations total {sum(t for t, _ in gen_diag):.1f} ms",
              file=sys.stderr)
        for i in slow:
            t, ex = gen_diag[i]
            print(f"[gen {i}] {t:.3f} ms (median {med:.3f}): " + "; ".join(
                f"{e.get('status')} c{e.get('cache_hit')} cm{e.get('compile_ms', 0):.1f} "
                f"d{(e.get('device_ms') or 0) * 1e3:.1f}us vc{e.get('verify_cached')}" for e in ex),
                file=sys.stderr)
    sec = max_over_ranks(local_sec)
    trials_per_s = trials / sec if sec > 0 else 0.0
    best_at_timed = engine.best().fitness if engine.archive else 0.0
    trials_at_timed = len(recorder.records)

    # ---------------- the rest of the search budget (untimed): best within
    # `budget` trials, the north star's "within 500 trials"
    while len(recorder.records) < budget:
        if generation(engine, recorder) == 0:
            break
    records = recorder.records
    best = engine.best()
    healthy = not poisoned()        # the measurements below need this process's context

    # ---------------- confirm the best instance: re-time the top distinct
    # instances (noise must not decide between near-equal kernels)
    confirmed = local_ev.confirm_top(k=10, reps=100, rounds=5) if best.fitness > 0 and healthy else []

    # ---------------- e2e: the same generations (a fresh engine, same seed:
    # warm-ups untimed, then the K timed ones) through the public API, with
    # the operands uploaded from pinned host memory every generation -- so
    # every trial is verified again, against a reference recomputed from the
    # uploaded operands -- and the verification results read back
    e2e = None
    if not args.no_e2e and healthy:
        # a freshly prepared operand too: nothing the main search learnt on
        # the device (verified instances, the straggler rule's fastest
        # launch) carries over into the replayed generations
        from paper_2006_05664_b200.evaluator import _op_args

        main_op = local_ev.op
        op = local_ev.op = local_ev.dev.prepare(dtype=settings.dtype, seed=settings.seed, **_op_args(spec))
        pa, pb = capi.PinnedBuffer(op.a_bytes), capi.PinnedBuffer(op.b_bytes)
        # stage the device operands in pinned host memory once (untimed)
        op.read_inputs(pa.ptr, pb.ptr)

        def upload():
            op.upload(pa.ptr, pb.ptr)

        e_engine, e_rec = new_search(RHO * (args.warmup + args.steps))
        for g in range(args.warmup):
            flush()
            generation(e_engine, e_rec, upload, replay=history[g])
        gc.collect()
        gc.disable()
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        e2e_trials = 0
        e_diag = [] if os.environ.get("OPEVO_BENCH_GEN_TIMES") == "1" else None
        for g in range(args.warmup, args.warmup + args.steps):
            flush()
            tg = time.perf_counter()
            e2e_trials += generation(e_engine, e_rec, upload, replay=history[g])
            if e_diag is not None:
                e_diag.append(1e3 * (time.perf_counter() - tg))
        barrier()
        f1.record()
        torch.cuda.synchronize()
        gc.enable()
        e_sec = max_over_ranks(f0.elapsed_time(f1) / 1e3)
        if e_diag is not None:
            print("[e2e gen ms] " + " ".join(f"{t:.2f}" for t in e_diag), file=sys.stderr)
        e2e = {"value": e2e_trials / e_sec if e_sec > 0 else 0.0, "unit": "trials/s",
               "h2d_bytes_per_step": (op.a_bytes + op.b_bytes) * world,
               "d2h_bytes_per_step": 16 * RHO, "steps": args.steps,
               "what": "the timed region's generations replayed -- a fresh engine with the same "
                       "seed told the recorded fitness asks the same configurations, each "
                       "measured again -- through GpuEvaluator.evaluate + OpEvo ask/tell on a "
                       "freshly prepared operand, operands uploaded from pinned host memory "
                       "every generation (reference recomputed, every trial re-verified), "
                       "compare results read back"}
        pa.close()
        pb.close()
        local_ev.op = main_op
        op.close()

    # ---------------- best kernel: re-time live (roofline.achieved)
    pk = peaks()
    roof = None
    best_knobs = None
    best_cold = None
    best_conf = confirmed[0] if confirmed else None
    if best_conf is not None:
        best_knobs = tuple(best_conf["knobs"])
        k = local_ev.dev.kernel(local_ev.op, best_knobs)
        # the kernel timed alone, as a burst: 100 back-to-back launches, or
        # fewer for long kernels so the graph lasts ~1 ms (9 ms of 4096^3
        # launches already runs into the board's power limit, and the
        # roofline denominator is the burst peak)
        est = confirmed[0]["ms"] if confirmed and confirmed[0].get("ms") else 0.0
        reps_graph = 100 if est <= 0.01 else max(5, min(100, int(1.0 / est)))
        ms = k.time(warmup=5, reps=reps_graph, flush_l2=False)
        ms_cold = k.time(warmup=2, reps=20, flush_l2=True)
        best_cold = spec.flops() / (ms_cold * 1e-3) / 1e12
        k.close()
        ach = spec.flops() / (ms * 1e-3) / 1e12
        peak = _dtype_peak(args.dtype, pk)
        nbytes = algo_bytes(spec, 2 if args.dtype == "bf16" else 4)
        ncu_op = ("" if args.dtype == "bf16" else args.dtype + ":") + args.op
        if args.dtype == "bf16" and spec.flops() / nbytes < pk["tflops"] * 1e3 / pk["hbm_gbs"]:
            # below the ridge (BMM 960x128x64x128: AI 32): HBM-bound roofline,
            # measured with the operands coming from HBM -- back-to-back
            # launches cycling over operand copies that together span more
            # than 2x the L2 (every launch's operands were evicted since their
            # last use); the single-launch cold figure (L2 flushed before each
            # launch) and the L2-warm figure the fitness uses ride along
            ms_rot, ncopies = hbm_fed_time(local_ev, spec, settings, best_knobs, nbytes)
            gbs = nbytes / (ms_rot * 1e-3) / 1e9
            roof = {"bound": "hbm", "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                    "frac": gbs / pk["hbm_gbs"], "traffic": _ncu_traffic(ncu_op, best_knobs),
                    "peak_source": f"{pk['source']} HBM copy bandwidth (MEASURED_PEAKS.json)",
                    "kernel_ms": ms_rot,
                    "timing": (f"HBM-fed: {16 * ncopies} back-to-back launches in one CUDA graph cycling "
                               f"over {ncopies} operand copies ({ncopies * nbytes / 1e6:.0f} MB > 2x L2)"),
                    "per_launch_bytes": nbytes,
                    "single_launch_cold_l2": {"kernel_ms": ms_cold, "gbs": nbytes / (ms_cold * 1e-3) / 1e9},
                    "l2_warm": {"kernel_ms": ms, "gbs": nbytes / (ms * 1e-3) / 1e9, "tflops": ach}}
        else:
            peak_src = _dtype_peak_source(args.dtype, pk)
            roof = {"bound": "fp32-fma" if args.dtype == "f32" else "tensor", "achieved": ach,
                    "peak": peak, "unit": "TFLOP/s",
                    "frac": ach / peak, "traffic": _ncu_traffic(ncu_op, best_knobs),
                    "peak_source": peak_src,
                    "kernel_ms": ms, "timing": f"{reps_graph} back-to-back launches in one CUDA graph"
                                               f" ({ms * reps_graph:.2f} ms: a burst)",
                    "per_launch_flops": spec.flops(), "per_launch_bytes": nbytes}

    # ---------------- cold kernel cache: a fresh evaluator over an empty
    # cubin cache (every instance NVRTC-compiled on the host pool), a few
    # generations of a fresh search
    cold = None
    if not args.no_cold and rank == 0 and world == 1 and healthy:
        cold = cold_cache_record(spec, space, settings, local, args)

    if rank == 0:
        cpu = None if (args.no_cpu or world > 1) else cpu_reference_arm(args.op, budget, args.seed)
        if cpu is not None:
            # §8d (2): the operator itself on the host cores, beside best_tflops
            cpu["operator"] = cpu_operator_throughput(args.op, "bf16" if args.dtype == "bf16" else "f32")
        if args.log:
            from paper_2006_05664_b200.logs import write_trial_log

            write_trial_log(args.log, records)
        best_tflops = best_conf["tflops"] if best_conf else 0.0
        line = {
            "metric": METRIC, "value": trials_per_s, "unit": "trials/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sec / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": args.dtype, "data": "synthetic",
            "config": {"workload": (f"OpEvo tuning of the sm_100a tcgen05 kernel family on {args.op} "
                                    f"bf16" if args.dtype == "bf16" else
                                    f"OpEvo tuning of the sm_100a tcgen05 3xTF32 family on {args.op} "
                                    f"fp32" if args.dtype == "tf32x3" else
                                    f"OpEvo tuning of the sm_100a fp32 SIMT family (paper TVM dense "
                                    f"schedule) on {args.op} fp32")
                                   + (" (BASELINE configs[1])" if args.op == DEFAULT_OP
                                      and args.dtype == "bf16" else ""),
                       "operator": args.op, "rho": RHO, "lambda": RHO, "q": 0.5,
                       "seed": args.seed, "trials_timed": trials, "search_budget": budget,
                       "ask": "python" if args.python_ask else "native (csrc/search.cpp)",
                       "space": ("reference operator space (fp32 SIMT family)" if args.dtype == "f32"
                                 else "reference operator space + stages (mapping.py)"),
                       "fitness_timing": fitness_timing(args, settings),
                       "l2_between_steps": "flushed: a 256 MB read pass (2x L2, leaves only clean "
                                           "lines) before every timed step",
                       "parallelism": f"trial sharding x{world}",
                       "kernel_cache": ("prebuilt cubins (build()); the operator's cached family "
                                        "loaded into the context and launched once before timing" if not args.no_preload
                                        else "prebuilt cubins (build()), loaded on first use")},
            "best_tflops": best_tflops,
            "best_frac_of_peak": best_tflops / _dtype_peak(args.dtype, pk),
            "best_knobs": list(best_knobs) if best_knobs else None,
            "best_confirmed": confirmed,
            "best_search_fitness": best.fitness,
            "best_config": space.config_to_json(best.config) if best.fitness > 0 else None,
            "best_tflops_at_timed_end": {"trials": trials_at_timed, "tflops": best_at_timed},
            "best_tflops_at_500_trials": best_tflops if len(records) >= 500 else None,
            "best_tflops_cold_l2": best_cold,
            "trials_to_95pct": trials_to_fraction(records),
            "wallclock_to_95pct_s": wallclock_to_fraction(records) / 1e3,
            "valid_fraction": sum(r.fitness > 0 for r in records) / len(records),
            "trials_total": len(records), "wall_s_timed": wall,
            "timed_trial_mix": {"trials": trials, "valid": tally["valid"],
                                "verified": tally["verified"],
                                "distinct_instances": len(tally["instances"]),
                                "valid_trials_per_s": tally["valid"] / sec if sec > 0 else 0.0,
                                "verified_trials_per_s": tally["verified"] / sec if sec > 0 else 0.0},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": tally["launches"],
            "cold_kernel_cache": cold,
            "timing": timing,
            "faulted_trials": sum(1 for r in records if (r.extra or {}).get("status") == "fault"),
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        evaluator.close()
        xchg.close()
    local_ev.close()
    if world > 1:
        dist.destroy_process_group()


def cold_cache_record(spec, space, settings, device: int, args, budget: int = 500,
                      max_s: float = 40.0) -> dict:
    """trials/s with an EMPTY cubin cache: a fresh
    evaluator compiles every instance it meets with NVRTC on a host pool of
    os.cpu_count() threads; a fresh search (same seed) runs `budget` trials
    or `max_s` seconds, wall-clock timed (compilation is host work).  The
    first generations are mostly infeasible configurations (nothing to
    compile), so a short run would overstate the cold rate."""
    import dataclasses
    import shutil
    import tempfile

    from paper_2006_05664_b200 import EngineConfig, OpEvo
    from paper_2006_05664_b200.evaluator import GpuEvaluator

    tmp = tempfile.mkdtemp(prefix="opevo_cold_cache_")
    threads = os.cpu_count() or 1
    cs = dataclasses.replace(settings, cache_dir=tmp, preload_family=False, compile_threads=threads)
    ev = GpuEvaluator(spec, space, device, cs)
    try:
        eng = OpEvo(space, EngineConfig(seed=args.seed, budget=budget, parents=RHO, offspring=RHO))
        trials = 0
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < max_s:
            asked = eng.ask()
            if not asked.configs:
                break
            eng.tell(list(zip(asked.configs, ev.evaluate(asked.configs))))
            trials += len(asked.configs)
        wall = time.perf_counter() - t0
        return {"value": trials / wall if wall > 0 else 0.0, "unit": "trials/s", "trials": trials,
                "wall_s": wall, "instances_compiled": len(os.listdir(tmp)),
                "nvrtc_pool_threads": threads, "timing": "host wall clock (NVRTC is host work)",
                "valid_trials": sum(h.status == "ok" for h in ev.history),
                "best_tflops": max((h.fitness for h in ev.history), default=0.0)}
    finally:
        ev.close()
        shutil.rmtree(tmp, ignore_errors=True)


def fitness_timing(args, settings) -> str:
    """How the search's fitness launches are timed (the bench line's config)."""
    if args.l2 == "cold":
        how = (f"{settings.reps} launches, each after a 2x-L2 read pass and timed alone (HBM-bound "
               f"operator: the fitness is its launch with the operands coming from HBM)")
    elif args.timing == "graph":
        how = f"{settings.reps} back-to-back launches in one CUDA graph, L2 warm (operands fit in L2)"
    else:
        how = (f"{settings.reps} back-to-back stream launches released by a device gate, L2 warm "
               f"(operands fit in L2)")
    return (how + f"; {settings.warmup} warm-up launches incl. the verified one; a "
            f"{settings.budget_ms} ms device budget per trial caps the repetitions, a candidate whose "
            f"verified launch alone exceeds it is timed by that launch, and one slower than "
            f"{settings.loser_ratio}x the fastest verified one gets {settings.loser_reps} launches")


def hbm_fed_time(ev, spec, settings, knobs, nbytes: int, l2_bytes: int = 126 << 20) -> tuple[float, int]:
    """ms per launch of `knobs` with its operands streamed from HBM: the
    instance bound to n freshly prepared operand copies (n x bytes > 2x L2,
    n >= 3) and launched back to back, cycling over them
    (capi.time_rotating)."""
    from paper_2006_05664_b200 import capi
    from paper_2006_05664_b200.evaluator import _op_args

    n = max(3, -(-2 * l2_bytes // nbytes) + 1)
    ops = [ev.dev.prepare(dtype=settings.dtype, seed=settings.seed + 1 + i, **_op_args(spec)) for i in range(n)]
    ks = []
    try:
        ks = [ev.dev.kernel(o, knobs) for o in ops]
        ms = min(capi.time_rotating(ks, warmup=1, reps=16 * n) for _ in range(3))
    finally:
        for k in ks:
            k.close()
        for o in ops:
            o.close()
    return ms, n


def _dtype_peak(dtype: str, pk: dict) -> float:
    """Roofline denominator (TFLOP/s of useful work) for a compute dtype."""
    if dtype == "bf16":
        return pk["tflops"]
    if dtype == "tf32x3":
        # kind::tf32 runs at half the bf16 rate and every K step issues three
        return pk["tflops"] / 2 / 3
    return FP32_PEAK


def _dtype_peak_source(dtype: str, pk: dict) -> str:
    if dtype == "bf16":
        return f"{pk['source']} burst bf16 (MEASURED_PEAKS.json)"
    if dtype == "tf32x3":
        return (f"{pk['source']} burst bf16 (MEASURED_PEAKS.json) / 2 (tf32 rate) / 3 (MMAs per "
                f"K step): the 3xTF32 ceiling in useful fp32 FLOP/s")
    return "nominal fp32 FMA peak at 1965 MHz (no measured figure)"


def algo_bytes(spec, elem: int) -> int:
    """Algorithmic bytes of one launch: every input read once, the output
    written once."""
    from paper_2006_05664_b200.operators import BatchMatMulSpec, MatMulSpec
    if isinstance(spec, MatMulSpec):
        return elem * (spec.n * spec.k + spec.m * spec.k + spec.n * spec.m)
    if isinstance(spec, BatchMatMulSpec):
        return elem * spec.b * (spec.n * spec.k + spec.m * spec.k + spec.n * spec.m)
    return elem * (spec.batch * spec.in_channels * spec.in_height * spec.in_width
                   + spec.out_channels * spec.in_channels * spec.kernel_h * spec.kernel_w
                   + spec.batch * spec.out_channels * spec.out_height * spec.out_width)


def _ncu_traffic(op: str, knobs) -> float | None:
    """DRAM read+write bytes per launch of this exact instance on this
    operator from the committed ncu capture (profiles/ncu_summary.json,
    keyed "operator|knobs", the operator prefixed "tf32x3:" / "f32:" for the
    fp32 families), else None."""
    path = os.path.join(REPO, "profiles", "ncu_summary.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
    except (OSError, ValueError):
        return None
    kernels = d.get("kernels", {})
    knobs = list(knobs)
    entry = kernels.get(op + "|" + ",".join(map(str, knobs)))
    if entry is None and len(knobs) == 14 and knobs[13] == 0:
        # captures taken before the conv `line` slot (ABI 6) carry 13 knobs;
        # line = 0 is the same kernel
        entry = kernels.get(op + "|" + ",".join(map(str, knobs[:13])))
    return entry.get("dram_bytes") if entry else None


if __name__ == "__main__":
    main()
