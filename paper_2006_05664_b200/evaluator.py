"""The B200 trial evaluator behind the reference's objective contract.

``make_gpu_objective(spec)`` returns ``(space, objective)`` exactly like the
reference's ``make_objective`` (``pkg/src/topotune/benchmarks.py:294-302``),
but the objective compiles, verifies and times a hand-written sm_100a kernel
through ``libopevo.so`` and returns measured TFLOP/s.  ``GpuEvaluator`` also
offers the batch interface the engine's ``run(..., evaluator=...)`` hook
takes (the reference's ``evaluate_batch`` seam, ``engine.py:264-290``):
kernels of a batch are NVRTC-compiled in parallel on host threads, then
launched one after another on the device.

Error semantics (reference ``engine.py:276-285``): an infeasible mapping, a
compile or launch failure, or an output that differs from the reference
scores 0; a missing device/driver/NVRTC raises ``FatalEvaluationError``; a
sticky context fault raises :class:`WorkerFault` so a scheduler can replace
the worker process.  There is no CPU fallback.
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

from . import capi
from .engine import FatalEvaluationError
from .mapping import FAMILY_CONV, config_to_knobs, gpu_operator_space
from .operators import BatchMatMulSpec, Conv2dSpec, MatMulSpec, OperatorSpec
from .spaces import SearchSpace

BF16_TOL = 1e-2
F32_TOL = 1e-4
# ABI dtype -> the name the mapping / space use
DTYPE_NAMES = {capi.BF16: "bf16", capi.F32: "f32", capi.F32_TF32X3: "tf32x3"}
DTYPES = {v: k for k, v in DTYPE_NAMES.items()}


class WorkerFault(FatalEvaluationError):
    """The CUDA context is poisoned; the worker process must be replaced."""


@dataclass
class EvalSettings:
    warmup: int = 3
    reps: int = 20
    flush_l2: int = 2             # timing mode: 0 graph, 1 cold L2, 2 gated stream (capi)
    seed: int = 1234
    compile_threads: int = 0          # 0 -> min(8, cpu count)
    cache_dir: str = capi.DEFAULT_CACHE
    dtype: int = capi.BF16
    # per-trial device budget (ms) and the straggler rule: a verified
    # candidate whose one-launch time exceeds loser_ratio x the fastest one
    # verified so far gets loser_reps timed launches (opevo_ctx_set_timing);
    # 1.2 rather than 1.5: same search outcomes over 8-16 seeds per operator,
    # 10-20 % more trials/s (profiles/round2/loser_ratio.txt)
    budget_ms: float = 0.3
    loser_ratio: float = 1.2
    loser_reps: int = 5
    # load every already-compiled instance of the operator's kernel family
    # into the context up front (a tuning service keeps them resident), so a
    # trial never pays a module load; uncached instances still compile/load
    # on demand
    preload_family: bool = False
    # ... and launch each of them once (a service's resident kernels are
    # warm too): a function's first launch in a process costs extra driver
    # and device time that is no property of the kernel
    warm_family: bool = False


@dataclass
class TrialInfo:
    fitness: float
    status: str
    knobs: tuple | None = None
    ms: float = 0.0
    rel_err: float = 0.0
    compile_ms: float = 0.0
    cache_hit: int = 0
    message: str = ""
    launches: int = 0
    verify_cached: int = 0        # 1: instance verified by an earlier trial on these operands
    extra: dict = field(default_factory=dict)

    def as_extra(self, gpu: int) -> dict:
        d = {"status": self.status, "device_ms": self.ms, "compile_ms": self.compile_ms,
             "rel_err": self.rel_err, "gpu_id": gpu, "cache_hit": self.cache_hit,
             "launches": self.launches, "verify_cached": self.verify_cached}
        if self.knobs is not None:
            d["knobs"] = list(self.knobs)
        if self.message:
            d["message"] = self.message[:200]
        return d


def _op_args(spec: OperatorSpec) -> dict:
    if isinstance(spec, MatMulSpec):
        return {"kind": capi.MATMUL, "rows": spec.n, "cols": spec.m, "depth": spec.k}
    if isinstance(spec, BatchMatMulSpec):
        return {"kind": capi.BATCHMATMUL, "batch": spec.b, "rows": spec.n, "cols": spec.m,
                "depth": spec.k}
    if isinstance(spec, Conv2dSpec):
        return {"kind": capi.CONV2D, "conv": [spec.batch, spec.in_channels, spec.in_height,
                                              spec.in_width, spec.out_channels, spec.kernel_h,
                                              spec.kernel_w, spec.stride, spec.padding]}
    raise TypeError(f"unknown operator spec: {spec!r}")


class GpuEvaluator:
    """Objective + batch evaluator bound to one operator on one B200."""

    def __init__(self, spec: OperatorSpec, space: SearchSpace | None = None, device: int = 0,
                 settings: EvalSettings | None = None, dev: "capi.Device | None" = None):
        self.spec = spec
        self.settings = settings or EvalSettings()
        self.dtype = DTYPE_NAMES[self.settings.dtype]
        self.space = space if space is not None else gpu_operator_space(spec, self.dtype)
        self.device_index = device
        self.tol = F32_TOL if self.settings.dtype in capi.FP32_OUT else BF16_TOL
        # `dev`: share an existing context (its loaded kernel modules); this
        # evaluator then owns only its operand, verification record and
        # timing state (the projection tool runs one per simulated rank)
        self._owns_dev = dev is None
        try:
            self.dev = dev if dev is not None else capi.Device(device, self.settings.cache_dir)
            self.op = self.dev.prepare(dtype=self.settings.dtype, seed=self.settings.seed,
                                       **_op_args(spec))
            self.dev.set_timing(self.settings.budget_ms, self.settings.loser_ratio,
                                self.settings.loser_reps)
        except (OSError, capi.OpevoError) as err:
            raise FatalEvaluationError(f"B200 evaluator unavailable: {err}") from err
        self.flops = float(spec.flops())
        self.last_extras: list[dict] = []
        self.history: list[TrialInfo] = []
        nthreads = self.settings.compile_threads or min(8, os.cpu_count() or 1)
        self._pool = ThreadPoolExecutor(max_workers=nthreads)
        self._staged: set = set()          # kernels already loaded in this context
        if self.settings.preload_family and self.dtype in ("bf16", "tf32x3"):
            self.preload_family()

    def close(self) -> None:
        self._pool.shutdown(wait=False)
        if getattr(self, "op", None) is not None:
            self.op.close()
            self.op = None
        if getattr(self, "dev", None) is not None:
            if getattr(self, "_owns_dev", True):
                self.dev.close()
            self.dev = None

    # -- the reference objective contract -----------------------------------
    def __call__(self, config: tuple) -> float:
        return self.evaluate([config])[0]

    # -- batch interface (engine.run evaluator hook) ----------------------------
    def evaluate(self, configs: list[tuple]) -> list[float]:
        infos = self.evaluate_infos(configs)
        self.last_extras = [i.as_extra(self.device_index) for i in infos]
        return [i.fitness for i in infos]

    def precompile(self, mapped) -> None:
        """Stage the distinct kernels of a batch on the host pool: NVRTC
        compile (or cubin-cache read) and module load into this device's
        context, in parallel, so the trials themselves only bind and launch."""
        distinct = {}
        for m in mapped:
            key = (m.family, m.batched, m.knobs.compile_key()) if m.valid else None
            if key is not None and key not in self._staged:
                distinct[key] = m

        def build(m):
            # failures are reported again (with status) by the trial itself
            self.dev.preload(self.op, m.knobs.as_tuple())

        if len(distinct) == 1:
            build(next(iter(distinct.values())))
        elif distinct:
            list(self._pool.map(build, distinct.values()))
        self._staged.update(distinct)

    def preload_family(self) -> int:
        """Load the cached instances reachable from this operator's space
        (prebuild.family_instances) into the context on the host pool.
        Returns how many were loaded."""
        from .prebuild import family_instances

        from .mapping import Knobs

        todo = []
        have = set(os.listdir(self.settings.cache_dir)) if os.path.isdir(self.settings.cache_dir) else set()
        for fam, batched, kn in family_instances(self.spec, self.dtype):
            if capi.kernel_key(fam, kn, batched, self.dtype == "tf32x3") + ".cubin" in have:
                todo.append((fam, batched, kn))

        def load(item):
            return self.dev.preload(self.op, item[2])[0] == capi.OK

        oks = list(self._pool.map(load, todo))
        # loaded modules need no staging when a batch first maps to them
        for (fam, batched, kn), ok in zip(todo, oks):
            if ok:
                self._staged.add((fam, bool(batched),
                                  Knobs(*kn, family=fam, batched=int(batched)).compile_key()))
        # (not under fault injection: a trapping instance must fault inside
        # a trial, where the isolation path handles it)
        if self.settings.warm_family and not os.environ.get("OPEVO_FAULT_KNOBS"):
            for (_fam, _batched, kn), ok in zip(todo, oks):
                if not ok:
                    continue
                try:
                    k = self.dev.kernel(self.op, kn)
                except capi.OpevoError:
                    continue                # infeasible on this operator (e.g. tiling)
                try:
                    k.run()
                finally:
                    k.close()
        return sum(oks)

    def evaluate_infos(self, configs: list[tuple]) -> list[TrialInfo]:
        """Map, stage (compile/load on the host pool) and measure a batch.
        The valid instances run as one ``opevo_trial_batch``: their checks and
        warm-ups are enqueued together, then their timed launches, so the
        host synchronises twice per batch rather than per trial."""
        mapped = [config_to_knobs(self.spec, self.space, c, self.dtype) for c in configs]
        self.precompile(mapped)
        valid = [m.knobs.as_tuple() for m in mapped if m.valid]
        s = self.settings
        try:
            trials = self.dev.trial_batch(self.op, valid, warmup=s.warmup, reps=s.reps,
                                          flush_l2=int(s.flush_l2), tol=self.tol) if valid else []
        except capi.OpevoError as err:
            if err.status == capi.ERR_STICKY:
                raise WorkerFault(f"device {self.device_index}: {err.message}") from err
            raise FatalEvaluationError(f"device {self.device_index}: {err.message}") from err
        it = iter(zip(valid, trials))
        out = []
        for m in mapped:
            if not m.valid:
                out.append(TrialInfo(0.0, "invalid_config", None, message=m.reason))
                continue
            knobs, t = next(it)
            out.append(self._info(knobs, t))
        self.history.extend(out)
        return out

    def confirm_top(self, k: int = 5, reps: int = 100, rounds: int = 5,
                    mode: int | None = None) -> list[dict]:
        """Re-time the ``k`` distinct kernel instances with the highest trial
        fitness seen so far, so that timing noise does not decide between
        near-equal instances.  Every instance is measured ``rounds`` times
        (``reps`` back-to-back launches each, rounds interleaved across the
        instances so drift hits all alike); the confirmed figure is the mean
        over rounds with its 95 % confidence half-width.  The archive (and
        with it the bit-exact trajectory) is untouched: this only decides
        which instance is reported as the best.  Returns one dict per
        instance, best confirmed first."""
        best: dict[tuple, float] = {}
        for info in self.history:
            if info.status == "ok" and info.knobs is not None and info.fitness > 0:
                best[info.knobs] = max(best.get(info.knobs, 0.0), info.fitness)
        top = sorted(best.items(), key=lambda kv: -kv[1])[:k]
        if not top:
            return []
        if mode is None:
            # the gated-stream fitness (mode 2) is confirmed as one CUDA graph
            # of back-to-back launches (mode 0): the kernel's own rate without
            # stream-launch gaps (~6 % at 1024^3, profiles/round2/
            # timing_modes.txt); a cold-L2 fitness (mode 1) is confirmed cold
            mode = 0 if int(self.settings.flush_l2) == 2 else int(self.settings.flush_l2)
        kernels = [self.dev.kernel(self.op, kn) for kn, _ in top]
        times: list[list[float]] = [[] for _ in top]
        # each measurement is a burst of ~1 ms at most (long kernels get
        # fewer launches): minutes of back-to-back 4096^3 launches would
        # measure the board's power limit, not the kernel
        nreps = [max(5, min(reps, int(1.0 / (self.flops / (fit * 1e9))))) if fit > 0 else reps
                 for _, fit in top]
        try:
            for _ in range(rounds):
                for i, kr in enumerate(kernels):
                    times[i].append(kr.time(warmup=3, reps=nreps[i], flush_l2=mode))
        finally:
            for kr in kernels:
                kr.close()
        # two-sided 95 % t quantiles for rounds - 1 degrees of freedom
        tq = {1: 12.706, 2: 4.303, 3: 3.182, 4: 2.776, 5: 2.571, 6: 2.447, 7: 2.365, 8: 2.306,
              9: 2.262}.get(rounds - 1, 1.96)
        out = []
        for (kn, fit), ts, n in zip(top, times, nreps):
            mean = sum(ts) / len(ts)
            sd = (sum((t - mean) ** 2 for t in ts) / (len(ts) - 1)) ** 0.5 if len(ts) > 1 else 0.0
            half = tq * sd / len(ts) ** 0.5
            out.append({"knobs": list(kn), "tflops": self.flops / (mean * 1e-3) / 1e12,
                        "ms": mean, "ci95_pct": 100.0 * half / mean if mean > 0 else None,
                        "search_tflops": fit, "rounds": rounds, "reps": n})
        out.sort(key=lambda d: -d["tflops"])
        return out

    def run_knobs(self, knobs: tuple) -> TrialInfo:
        """One trial through ``opevo_trial`` (the single-configuration path)."""
        s = self.settings
        t = self.dev.trial(self.op, knobs, warmup=s.warmup, reps=s.reps, flush_l2=s.flush_l2,
                           tol=self.tol)
        return self._info(knobs, t)

    def _info(self, knobs: tuple, t: "capi.Trial") -> TrialInfo:
        if t.status == capi.ERR_STICKY:
            raise WorkerFault(f"device {self.device_index}: {t.message}")
        if t.status < 0:
            raise FatalEvaluationError(f"device {self.device_index}: {t.message}")
        if t.status != capi.OK:
            return TrialInfo(0.0, capi.STATUS_NAMES.get(t.status, str(t.status)), knobs,
                             rel_err=t.rel_err, compile_ms=t.compile_ms, cache_hit=t.cache_hit,
                             message=t.message, launches=t.launches)
        fit = self.flops / (t.ms * 1e-3) / 1e12 if t.ms > 0 else 0.0
        if not math.isfinite(fit):
            fit = 0.0
        return TrialInfo(fit, "ok", knobs, ms=t.ms, rel_err=t.rel_err, compile_ms=t.compile_ms,
                         cache_hit=t.cache_hit, launches=t.launches, verify_cached=t.verify_cached)


def make_gpu_objective(spec: OperatorSpec, space: SearchSpace | None = None, device: int = 0,
                       settings: EvalSettings | None = None):
    """``(space, objective)`` with the objective measured on a B200 (TFLOP/s)."""
    ev = GpuEvaluator(spec, space, device, settings)
    return ev.space, ev
