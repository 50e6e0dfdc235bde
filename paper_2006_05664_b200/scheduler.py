"""Device-affine trial scheduling: one independent trial per GPU per slot.

Replaces the reference's ``evaluate_batch(objective, configs, concurrency)``
(``pkg/src/topotune/engine.py:264-290``), whose only parallelism is a thread
pool over one objective.  Trials are independent, so
there is no data-path collective: a batch is split by ask index round-robin
over devices, each device evaluates its share, and the fitnesses are
gathered back into ask order before ``tell`` (archive insertion is in ask
order regardless, ``engine.py:218-220``).

Two drivers:

* :class:`ShardedEvaluator` -- one process per GPU (``torchrun``); every rank
  runs an identical engine replica (same seed, same told fitnesses, so the
  same asks) and the only exchange is one small ``all_reduce`` of the
  per-trial result rows per generation.
* :class:`TrialScheduler` -- one controller process with a worker *process*
  per GPU.  A worker whose CUDA context is poisoned by a faulting candidate
  (``WorkerFault``) is replaced and the rest of its shard re-submitted; the
  faulting configuration scores 0, like any invalid configuration.
"""

from __future__ import annotations

import multiprocessing as mp
import traceback
from dataclasses import asdict

from .engine import FatalEvaluationError
from .evaluator import EvalSettings, GpuEvaluator, TrialInfo, WorkerFault
from .spaces import SearchSpace

# result row layout for the all-reduce
_COLS = ("fitness", "device_ms", "compile_ms", "rel_err", "status", "cache_hit", "gpu_id", "present",
         "launches")
_STATUS = ("ok", "invalid_config", "compile_error", "launch_error", "verify_failed", "fault")


def _status_code(name: str) -> int:
    return _STATUS.index(name) if name in _STATUS else len(_STATUS)


def shard_indices(n: int, world: int, rank: int) -> list[int]:
    """Round-robin by ask index: rank r evaluates configs r, r+W, r+2W, ..."""
    return list(range(rank, n, world))


class ShardedEvaluator:
    """Batch evaluator for ``run(..., evaluator=...)`` under torch.distributed."""

    def __init__(self, local: GpuEvaluator | None, rank: int, world: int, group=None,
                 device=None, local_fn=None):
        self.local = local
        self.local_fn = local_fn            # testing hook: configs -> list[TrialInfo]
        self.rank, self.world = rank, world
        self.group = group
        self.device = device                # torch device for the collective tensor
        self.last_extras: list[dict] = []

    def _local_infos(self, configs: list[tuple]) -> list[TrialInfo]:
        if self.local_fn is not None:
            return self.local_fn(configs)
        return self.local.evaluate_infos(configs)

    def __call__(self, configs: list[tuple]) -> list[float]:
        import torch
        import torch.distributed as dist

        mine = shard_indices(len(configs), self.world, self.rank)
        infos = self._local_infos([configs[i] for i in mine]) if mine else []
        rows = torch.zeros((len(configs), len(_COLS)), dtype=torch.float64)
        for i, info in zip(mine, infos):
            rows[i] = torch.tensor([info.fitness, info.ms, info.compile_ms, info.rel_err,
                                    _status_code(info.status), info.cache_hit, self.rank, 1.0,
                                    info.launches], dtype=torch.float64)
        if self.device is not None:
            rows = rows.to(self.device)
        dist.all_reduce(rows, group=self.group)
        rows = rows.cpu()
        if not bool((rows[:, 7] == 1.0).all()):
            raise FatalEvaluationError("a trial was evaluated by zero or several ranks")
        self.last_extras = []
        fits = []
        for r in rows.tolist():
            code = int(r[4])
            self.last_extras.append({"status": _STATUS[code] if code < len(_STATUS) else "error",
                                     "device_ms": r[1], "compile_ms": r[2], "rel_err": r[3],
                                     "cache_hit": int(r[5]), "gpu_id": int(r[6]),
                                     "launches": int(r[8])})
            fits.append(r[0])
        return fits


# ----------------------------------------------------------------------------
# process-pool scheduler
# ----------------------------------------------------------------------------

def _worker_main(conn, spec, space_json, device, settings_dict):
    try:
        space = SearchSpace.from_json(space_json)
        ev = GpuEvaluator(spec, space, device, EvalSettings(**settings_dict))
    except Exception as err:   # noqa: BLE001 - reported to the controller
        conn.send(("fatal", f"{type(err).__name__}: {err}"))
        return
    conn.send(("ready", device))
    while True:
        msg = conn.recv()
        if msg is None:
            break
        idx, config = msg
        try:
            info = ev.evaluate_infos([config])[0]
            conn.send(("result", idx, asdict(info)))
        except WorkerFault as err:
            conn.send(("fault", idx, str(err)))
            return
        except FatalEvaluationError as err:
            conn.send(("fatal", str(err)))
            return
        except Exception:   # noqa: BLE001
            conn.send(("error", idx, traceback.format_exc(limit=3)))
    ev.close()


class _Worker:
    def __init__(self, ctx, spec, space, device, settings):
        self.device = device
        self.args = (spec, space.to_json(), device, asdict(settings))
        self.ctx = ctx
        self.start()

    def start(self):
        self.conn, child = self.ctx.Pipe()
        self.proc = self.ctx.Process(target=_worker_main, args=(child, *self.args), daemon=True)
        self.proc.start()
        child.close()
        msg = self.conn.recv()
        if msg[0] != "ready":
            raise FatalEvaluationError(f"GPU worker {self.device} failed to start: {msg[1]}")

    def stop(self):
        try:
            self.conn.send(None)
        except (BrokenPipeError, OSError):
            pass
        self.proc.join(timeout=10)
        if self.proc.is_alive():
            self.proc.kill()


class TrialScheduler:
    """Evaluate batches over several GPUs with one worker process each."""

    def __init__(self, spec, space: SearchSpace, devices: list[int],
                 settings: EvalSettings | None = None):
        self.space = space
        self.settings = settings or EvalSettings()
        ctx = mp.get_context("spawn")
        self.workers = [_Worker(ctx, spec, space, d, self.settings) for d in devices]
        self.last_extras: list[dict] = []
        self.respawns = 0

    def close(self):
        for w in self.workers:
            w.stop()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __call__(self, configs: list[tuple]) -> list[float]:
        n = len(configs)
        results: list[dict | None] = [None] * n
        queues = [shard_indices(n, len(self.workers), r) for r in range(len(self.workers))]
        busy = {}
        for w, q in zip(self.workers, queues):
            if q:
                i = q.pop(0)
                w.conn.send((i, configs[i]))
                busy[w] = (i, q)
        while busy:
            ready = mp.connection.wait([w.conn for w in busy])
            for w in [w for w in list(busy) if w.conn in ready]:
                i, q = busy.pop(w)
                try:
                    msg = w.conn.recv()
                except EOFError:
                    msg = ("fault", i, "worker died")
                if msg[0] == "result":
                    results[i] = msg[2]
                elif msg[0] in ("fault", "error"):
                    results[i] = asdict(TrialInfo(0.0, "fault", message=str(msg[2])[:200]))
                    if msg[0] == "fault":
                        w.proc.join(timeout=10)
                        w.start()
                        self.respawns += 1
                else:
                    raise FatalEvaluationError(f"GPU worker {w.device}: {msg[1]}")
                if q:
                    j = q.pop(0)
                    w.conn.send((j, configs[j]))
                    busy[w] = (j, q)
        self.last_extras = []
        fits = []
        for i, r in enumerate(results):
            gpu = self.workers[i % len(self.workers)].device
            info = TrialInfo(**r)
            self.last_extras.append(info.as_extra(gpu))
            fits.append(info.fitness)
        return fits
