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
  per GPU, each running its whole shard as one trial-batch pipeline.  A
  worker whose CUDA context is poisoned by a faulting candidate
  (``WorkerFault``) is replaced and its shard re-run one configuration at a
  time; the faulting configuration scores 0, like any invalid one.

Both survive a faulting candidate: :class:`ShardedEvaluator` moves a rank
whose context was poisoned onto a worker process (:class:`ProcessEvaluator`)
and exchanges results over a host (gloo) group.
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
         "launches", "verify_cached", "abort")
_STATUS = ("ok", "invalid_config", "compile_error", "launch_error", "verify_failed", "fault")


def _status_code(name: str) -> int:
    return _STATUS.index(name) if name in _STATUS else len(_STATUS)


def shard_indices(n: int, world: int, rank: int) -> list[int]:
    """Round-robin by ask index: rank r evaluates configs r, r+W, r+2W, ..."""
    return list(range(rank, n, world))


# ----------------------------------------------------------------------------
# worker process: one GpuEvaluator, a whole shard per message
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
        try:
            if msg[0] == "batch":
                conn.send(("infos", [asdict(i) for i in ev.evaluate_infos(list(msg[1]))]))
            elif msg[0] == "flush":
                ev.dev.flush_l2()
                conn.send(("ok",))
            else:
                conn.send(("error", f"unknown request {msg[0]!r}"))
        except WorkerFault as err:
            conn.send(("fault", str(err)))
            return
        except FatalEvaluationError as err:
            conn.send(("fatal", str(err)))
            return
        except Exception:   # noqa: BLE001
            conn.send(("error", traceback.format_exc(limit=3)))
    ev.close()


class _Worker:
    """A GPU worker process.  ``evaluate`` sends a whole shard in one message
    (the process runs it as one ``opevo_trial_batch`` pipeline); when the
    shard faults -- a candidate poisoned the worker's CUDA context, and the
    batch does not say which -- the worker is replaced and the shard is
    re-run one configuration per message, so exactly the faulting
    candidates score 0 (status "fault", the reference's failure-to-0
    semantics, engine.py:276-285) and each costs one more respawn."""

    def __init__(self, ctx, spec, space, device, settings):
        self.device = device
        self.args = (spec, space.to_json(), device, asdict(settings))
        self.ctx = ctx
        self.respawns = 0
        self.start()

    def start(self):
        self.conn, child = self.ctx.Pipe()
        self.proc = self.ctx.Process(target=_worker_main, args=(child, *self.args), daemon=True)
        self.proc.start()
        child.close()
        msg = self.conn.recv()
        if msg[0] != "ready":
            raise FatalEvaluationError(f"GPU worker {self.device} failed to start: {msg[1]}")

    def respawn(self):
        self.proc.join(timeout=10)
        if self.proc.is_alive():
            self.proc.kill()
        self.start()
        self.respawns += 1

    def stop(self):
        try:
            self.conn.send(None)
        except (BrokenPipeError, OSError):
            pass
        self.proc.join(timeout=10)
        if self.proc.is_alive():
            self.proc.kill()

    def send_batch(self, configs: list[tuple]) -> None:
        self.conn.send(("batch", list(configs)))

    def _recv(self):
        try:
            return self.conn.recv()
        except EOFError:
            return ("fault", "worker died")

    def finish_batch(self, configs: list[tuple]) -> list[TrialInfo]:
        """Result of the batch sent with ``send_batch`` (isolating faults)."""
        msg = self._recv()
        if msg[0] == "infos":
            return [TrialInfo(**d) for d in msg[1]]
        if msg[0] == "fatal":
            raise FatalEvaluationError(f"GPU worker {self.device}: {msg[1]}")
        if msg[0] == "error":
            raise FatalEvaluationError(f"GPU worker {self.device}: {msg[1]}")
        # fault: replace the worker and find the faulting candidate(s)
        self.respawn()
        if len(configs) == 1:
            return [TrialInfo(0.0, "fault", message=str(msg[1])[:200])]
        out = []
        for c in configs:
            self.send_batch([c])
            out.extend(self.finish_batch([c]))
        return out

    def evaluate(self, configs: list[tuple]) -> list[TrialInfo]:
        self.send_batch(configs)
        return self.finish_batch(configs)

    def flush_l2(self) -> None:
        self.conn.send(("flush",))
        msg = self._recv()
        if msg[0] != "ok":
            if msg[0] == "fault":
                self.respawn()
            else:
                raise FatalEvaluationError(f"GPU worker {self.device}: {msg[1]}")


class ProcessEvaluator:
    """``GpuEvaluator``'s batch interface served by a worker process (a fresh
    CUDA context that a faulting candidate cannot take down with the caller)."""

    def __init__(self, spec, space: SearchSpace, device: int = 0,
                 settings: EvalSettings | None = None):
        self.device_index = device
        self.worker = _Worker(mp.get_context("spawn"), spec, space, device, settings or EvalSettings())
        self.last_extras: list[dict] = []
        self.history: list[TrialInfo] = []

    def evaluate_infos(self, configs: list[tuple]) -> list[TrialInfo]:
        infos = self.worker.evaluate(configs) if configs else []
        self.history.extend(infos)
        return infos

    def evaluate(self, configs: list[tuple]) -> list[float]:
        infos = self.evaluate_infos(configs)
        self.last_extras = [i.as_extra(self.device_index) for i in infos]
        return [i.fitness for i in infos]

    @property
    def respawns(self) -> int:
        return self.worker.respawns

    def flush_l2(self) -> None:
        self.worker.flush_l2()

    def close(self) -> None:
        self.worker.stop()


# ----------------------------------------------------------------------------
# one process per GPU (torchrun)
# ----------------------------------------------------------------------------

class ShmExchange:
    """Sum-all-reduce of the per-generation result table through POSIX shared
    memory, for the ranks of ONE node (bench.py's contract: N GPUs of one
    box).  A gloo all-reduce of the 8 x 11 fp64 table measured 1.4 ms at 2
    ranks and 29 ms at 8 on loopback TCP -- longer than a whole generation --
    while this takes microseconds and, like gloo, touches no CUDA context (a
    rank whose context a faulting candidate poisoned still takes part).

    Layout: per rank a 64-byte sequence slot, then two buffers (double
    buffering by generation parity) of [world][max_rows][cols] fp64.  A rank
    writes its rows into buffer gen % 2, publishes gen in its slot, waits for
    every slot to reach gen and sums the ranks' rows.  A rank cannot write
    buffer gen % 2 again (at gen + 2) before every rank has published gen + 1,
    which each does only after reading gen, so two buffers suffice.  Rows
    evaluated by one rank and zero elsewhere sum exactly.  A rank that stops
    publishing turns into a FatalEvaluationError after ``timeout_s``."""

    def __init__(self, path: str, rank: int, world: int, max_rows: int, cols: int,
                 create: bool = False, timeout_s: float = 120.0):
        import mmap

        import numpy as np

        self.rank, self.world, self.max_rows, self.cols = rank, world, max_rows, cols
        self.path, self.timeout_s = path, timeout_s
        self.gen = 0
        seq_bytes = 64 * world
        buf = world * max_rows * cols * 8
        size = seq_bytes + 2 * buf
        if create:
            with open(path, "wb") as fh:
                fh.truncate(size)
        self._fh = open(path, "r+b")
        self._mm = mmap.mmap(self._fh.fileno(), size)
        self.seq = np.ndarray((world, 8), dtype=np.int64, buffer=self._mm, offset=0)
        self.data = np.ndarray((2, world, max_rows, cols), dtype=np.float64, buffer=self._mm,
                               offset=seq_bytes)

    @classmethod
    def create(cls, rank: int, world: int, group=None, max_rows: int = 64, cols: int = len(_COLS),
               timeout_s: float = 120.0) -> "ShmExchange":
        """Rank 0 creates the segment; its name reaches the others through one
        object broadcast on ``group`` (setup only)."""
        import os
        import uuid

        import torch.distributed as dist

        name = [f"/dev/shm/opevo_xchg_{uuid.uuid4().hex}" if rank == 0 else None]
        if rank == 0:
            ex = cls(name[0], rank, world, max_rows, cols, create=True, timeout_s=timeout_s)
        dist.broadcast_object_list(name, src=0, group=group)
        if rank != 0:
            ex = cls(name[0], rank, world, max_rows, cols, timeout_s=timeout_s)
        dist.barrier(group=group)
        if rank == 0:
            os.unlink(name[0])          # the mappings stay valid; nothing is left behind
        return ex

    def allreduce(self, rows):
        """Sum of every rank's ``rows`` ([n][cols] fp64, n <= max_rows)."""
        import time

        import numpy as np

        n = rows.shape[0]
        if n > self.max_rows or rows.shape[1] != self.cols:
            raise ValueError(f"exchange holds {self.max_rows} x {self.cols} rows, got {rows.shape}")
        self.gen += 1
        b = self.gen & 1
        self.data[b, self.rank, :n] = rows
        self.seq[self.rank, 0] = self.gen            # publish (x86 stores stay in order)
        t0 = time.perf_counter()
        spins = 0
        while int(self.seq[:, 0].min()) < self.gen:
            spins += 1
            if spins > 2000:
                time.sleep(0.0001)
                if time.perf_counter() - t0 > self.timeout_s:
                    raise FatalEvaluationError(
                        f"rank exchange timed out at generation {self.gen}: a rank stopped")
        return np.asarray(self.data[b, :, :n].sum(axis=0))

    def barrier(self) -> None:
        import numpy as np

        self.allreduce(np.zeros((1, self.cols)))

    def max(self, x: float) -> float:
        import numpy as np

        # a max through the sum: every rank contributes one column of its own
        cols = np.zeros((1, self.cols))
        if self.world > self.cols:
            raise ValueError("too many ranks for max()")
        cols[0, self.rank] = x
        return float(self.allreduce(cols)[0, :self.world].max())

    def close(self) -> None:
        try:
            self._mm.close()
            self._fh.close()
        except (OSError, ValueError, BufferError):
            pass


class ShardedEvaluator:
    """Batch evaluator for ``run(..., evaluator=...)`` under torch.distributed.

    The per-generation exchange is one sum-all-reduce of a small host table,
    through :class:`ShmExchange` (``exchange``; the ranks of one node) or
    else ``torch.distributed`` over ``group`` (gloo) -- no CUDA context is
    involved either way, so a rank whose context a faulting candidate
    poisoned still takes part.  On such
    a fault (``WorkerFault``) the rank moves its evaluation to a worker
    process (:class:`ProcessEvaluator`, a fresh context), which re-runs the
    shard with the faulting candidate isolated and scored 0; the other ranks
    never notice.  A fatal error on any rank (no device, NVRTC missing) sets
    the row's abort flag and every rank raises it after the exchange, so no
    rank is left waiting in the collective."""

    def __init__(self, local: GpuEvaluator | None, rank: int, world: int, group=None,
                 device=None, local_fn=None, respawn=None, exchange: ShmExchange | None = None):
        self.local = local
        self.local_fn = local_fn            # testing hook: configs -> list[TrialInfo]
        self.rank, self.world = rank, world
        self.group = group
        self.device = device                # unused (kept for callers); the exchange is on host
        # () -> a replacement evaluator after a fault, e.g.
        # lambda: ProcessEvaluator(spec, space, device, settings)
        self.respawn = respawn
        self.exchange = exchange            # shared-memory exchange (else torch.distributed)
        self.fallback = None
        self.poisoned = False               # this process's CUDA context is unusable
        self.faults = 0
        self.last_extras: list[dict] = []

    def _local_infos(self, configs: list[tuple]) -> list[TrialInfo]:
        if self.fallback is not None:
            return self.fallback.evaluate_infos(configs)
        if self.local_fn is not None:
            return self.local_fn(configs)
        return self.local.evaluate_infos(configs)

    def flush_l2(self) -> None:
        if self.fallback is not None:
            self.fallback.flush_l2()
        elif self.local is not None and not self.poisoned:
            self.local.dev.flush_l2()

    def __call__(self, configs: list[tuple]) -> list[float]:
        import torch
        import torch.distributed as dist

        mine = shard_indices(len(configs), self.world, self.rank)
        abort_msg = ""
        infos: list[TrialInfo] = []
        try:
            infos = self._local_infos([configs[i] for i in mine]) if mine else []
        except WorkerFault as err:
            self.poisoned = True
            self.faults += 1
            if self.respawn is None:
                abort_msg = str(err)
            else:
                try:
                    self.fallback = self.respawn()
                    infos = self.fallback.evaluate_infos([configs[i] for i in mine])
                except FatalEvaluationError as err2:
                    abort_msg = str(err2)
        except FatalEvaluationError as err:
            abort_msg = str(err)
        rows = torch.zeros((len(configs), len(_COLS)), dtype=torch.float64)
        for i, info in zip(mine, infos):
            rows[i] = torch.tensor([info.fitness, info.ms, info.compile_ms, info.rel_err,
                                    _status_code(info.status), info.cache_hit, self.rank, 1.0,
                                    info.launches, info.verify_cached, 0.0], dtype=torch.float64)
        if abort_msg:
            rows[mine, 7] = 1.0
            rows[mine, 10] = 1.0 + self.rank
        if self.exchange is not None:
            rows = torch.from_numpy(self.exchange.allreduce(rows.numpy()))
        else:
            dist.all_reduce(rows, group=self.group)
        if bool((rows[:, 10] > 0).any()):
            culprit = int(rows[:, 10].max().item()) - 1
            raise FatalEvaluationError(f"rank {culprit} aborted the generation"
                                       + (f": {abort_msg}" if abort_msg else ""))
        if not bool((rows[:, 7] == 1.0).all()):
            raise FatalEvaluationError("a trial was evaluated by zero or several ranks")
        self.last_extras = []
        fits = []
        for r in rows.tolist():
            code = int(r[4])
            self.last_extras.append({"status": _STATUS[code] if code < len(_STATUS) else "error",
                                     "device_ms": r[1], "compile_ms": r[2], "rel_err": r[3],
                                     "cache_hit": int(r[5]), "gpu_id": int(r[6]),
                                     "launches": int(r[8]), "verify_cached": int(r[9])})
            fits.append(r[0])
        return fits

    def close(self) -> None:
        if self.fallback is not None:
            self.fallback.close()


# ----------------------------------------------------------------------------
# single controller, one worker process per GPU
# ----------------------------------------------------------------------------

class TrialScheduler:
    """Evaluate batches over several GPUs with one worker process each: every
    worker gets its round-robin shard as one message (one trial-batch
    pipeline per GPU), all shards run at once, results come back in ask
    order; a faulting shard is isolated and its worker replaced."""

    def __init__(self, spec, space: SearchSpace, devices: list[int],
                 settings: EvalSettings | None = None):
        self.space = space
        self.settings = settings or EvalSettings()
        ctx = mp.get_context("spawn")
        self.workers = [_Worker(ctx, spec, space, d, self.settings) for d in devices]
        self.last_extras: list[dict] = []

    @property
    def respawns(self) -> int:
        return sum(w.respawns for w in self.workers)

    def close(self):
        for w in self.workers:
            w.stop()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __call__(self, configs: list[tuple]) -> list[float]:
        n = len(configs)
        shards = [shard_indices(n, len(self.workers), r) for r in range(len(self.workers))]
        for w, idx in zip(self.workers, shards):
            if idx:
                w.send_batch([configs[i] for i in idx])
        results: list[TrialInfo | None] = [None] * n
        for w, idx in zip(self.workers, shards):
            if idx:
                for i, info in zip(idx, w.finish_batch([configs[i] for i in idx])):
                    results[i] = info
        self.last_extras = []
        fits = []
        for i, info in enumerate(results):
            self.last_extras.append(info.as_extra(self.workers[i % len(self.workers)].device))
            fits.append(info.fitness)
        return fits
