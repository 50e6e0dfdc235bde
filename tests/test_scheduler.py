"""Multi-rank trial sharding on CPU: world_size 2 over gloo.

Each rank runs an engine replica and evaluates its round-robin share of every
ask batch through a fake local evaluator; the all_reduce must reassemble the
fitnesses in ask order so that both replicas (and a single-process run) see
identical trajectories.
"""

import hashlib
import json
import os
import socket
import tempfile

import pytest
import torch.distributed as dist
import torch.multiprocessing as tmp

from paper_2006_05664_b200 import EngineConfig, MatMulSpec, run
from paper_2006_05664_b200.engine import FatalEvaluationError
from paper_2006_05664_b200.evaluator import TrialInfo, WorkerFault
from paper_2006_05664_b200.mapping import config_to_knobs, gpu_operator_space
from paper_2006_05664_b200.scheduler import ShardedEvaluator, ShmExchange, shard_indices

SPEC = MatMulSpec(1024, 1024, 1024)


def fake_infos(space, rank):
    def local(cfgs):
        out = []
        for c in cfgs:
            m = config_to_knobs(SPEC, space, c)
            if not m.valid:
                out.append(TrialInfo(0.0, "invalid_config"))
                continue
            h = hashlib.sha256(repr(c).encode()).digest()
            out.append(TrialInfo(1 + h[0] / 2.55, "ok", m.knobs.as_tuple(), ms=0.01 * (rank + 1)))
        return out
    return local


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir, shm=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    space = gpu_operator_space(SPEC)
    xchg = ShmExchange.create(rank, world) if shm else None
    ev = ShardedEvaluator(None, rank, world, local_fn=fake_infos(space, rank), exchange=xchg)
    best, recs = run(space, EngineConfig(seed=5, budget=96), None, evaluator=ev)
    with open(os.path.join(out_dir, f"r{rank}.json"), "w") as fh:
        json.dump({"seq": [[r.config, r.fitness] for r in recs],
                   "gpus": [r.extra["gpu_id"] for r in recs]}, fh)
    dist.destroy_process_group()


def test_shard_indices_partition():
    for n in (1, 7, 8, 13):
        for w in (1, 2, 4, 8):
            got = sorted(i for r in range(w) for i in shard_indices(n, w, r))
            assert got == list(range(n))


@pytest.mark.parametrize("shm", [False, True])
def test_two_rank_gloo_sharding_matches_single_process(shm):
    """Through a gloo all-reduce and through the shared-memory exchange."""
    space = gpu_operator_space(SPEC)
    # single-process reference trajectory with the same fitness function
    local = fake_infos(space, 0)
    _, single = run(space, EngineConfig(seed=5, budget=96), lambda c: local([c])[0].fitness)
    with tempfile.TemporaryDirectory() as d:
        tmp.start_processes(_worker, args=(2, _free_port(), d, shm), nprocs=2, start_method="spawn")
        r0 = json.load(open(os.path.join(d, "r0.json")))
        r1 = json.load(open(os.path.join(d, "r1.json")))
    want = [[r.config, r.fitness] for r in single]
    assert r0["seq"] == r1["seq"] == want
    # ask index i was evaluated by rank i % 2 within every generation of 8
    assert r0["gpus"][:8] == [0, 1] * 4


class _Replacement:
    """Stands in for the worker process a faulted rank moves to: it scores
    the trial that faulted 0 (status fault) and evaluates the rest."""

    def __init__(self, space, rank, bad):
        self.inner, self.bad, self.calls = fake_infos(space, rank), bad, 0

    def evaluate_infos(self, cfgs):
        self.calls += 1
        return [TrialInfo(0.0, "fault") if c == self.bad else self.inner([c])[0] for c in cfgs]


def _fault_worker(rank, world, port, out_dir, mode):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    space = gpu_operator_space(SPEC)
    state = {"gen": 0, "bad": None}
    inner = fake_infos(space, rank)

    def local(cfgs):
        state["gen"] += 1
        if rank == 1 and state["gen"] == 3:
            state["bad"] = cfgs[0]
            if mode == "fault":
                raise WorkerFault("device 1: unspecified launch failure (injected)")
            raise FatalEvaluationError("no NVRTC (injected)")
        return inner(cfgs)

    repl = {}
    ev = ShardedEvaluator(None, rank, world, local_fn=local, exchange=ShmExchange.create(rank, world),
                          respawn=lambda: repl.setdefault("r", _Replacement(space, rank, state["bad"])))
    result = {}
    try:
        best, recs = run(space, EngineConfig(seed=5, budget=96), None, evaluator=ev)
        result = {"ok": True, "seq": [[r.config, r.fitness] for r in recs],
                  "status": [r.extra["status"] for r in recs], "poisoned": ev.poisoned,
                  "fallback_calls": repl["r"].calls if "r" in repl else 0}
    except FatalEvaluationError as err:
        result = {"ok": False, "error": str(err)}
    with open(os.path.join(out_dir, f"r{rank}.json"), "w") as fh:
        json.dump(result, fh)
    dist.destroy_process_group()


def test_two_rank_fault_is_isolated_on_the_faulting_rank():
    """Rank 1's context is poisoned in generation 3: it moves to a
    replacement evaluator, the faulting trial scores 0 (status fault), both
    replicas keep identical trajectories and the run completes."""
    with tempfile.TemporaryDirectory() as d:
        tmp.start_processes(_fault_worker, args=(2, _free_port(), d, "fault"), nprocs=2,
                            start_method="spawn")
        r0 = json.load(open(os.path.join(d, "r0.json")))
        r1 = json.load(open(os.path.join(d, "r1.json")))
    assert r0["ok"] and r1["ok"]
    assert r0["seq"] == r1["seq"] and len(r0["seq"]) == 96
    assert r0["status"].count("fault") == 1 and r0["status"][17] == "fault"
    assert r1["poisoned"] and r1["fallback_calls"] >= 1 and not r0["poisoned"]


def test_two_rank_fatal_error_aborts_every_rank_together():
    """A fatal error on one rank raises FatalEvaluationError on every rank
    after the exchange -- nobody is left waiting in the collective."""
    with tempfile.TemporaryDirectory() as d:
        tmp.start_processes(_fault_worker, args=(2, _free_port(), d, "fatal"), nprocs=2,
                            start_method="spawn")
        r0 = json.load(open(os.path.join(d, "r0.json")))
        r1 = json.load(open(os.path.join(d, "r1.json")))
    assert not r0["ok"] and not r1["ok"]
    assert "rank 1" in r0["error"] and "no NVRTC" in r1["error"]


def _xchg_worker(rank, world, port, out_dir):
    import numpy as np

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ex = ShmExchange.create(rank, world)
    res = []
    for g in range(200):                       # generations of different sizes
        n = 1 + (g % 8)
        rows = np.zeros((n, ex.cols))
        rows[rank::world] = g + rank + 0.5
        res.append(ex.allreduce(rows)[:, 0].tolist())
    res.append([ex.max(float(rank * 3))])
    with open(os.path.join(out_dir, f"x{rank}.json"), "w") as fh:
        json.dump(res, fh)
    ex.close()
    dist.destroy_process_group()


def test_shm_exchange_four_ranks():
    """Every rank sees every rank's rows summed, generation after generation
    (double buffering by parity), and the max over ranks."""
    world = 4
    with tempfile.TemporaryDirectory() as d:
        tmp.start_processes(_xchg_worker, args=(world, _free_port(), d), nprocs=world, start_method="spawn")
        got = [json.load(open(os.path.join(d, f"x{r}.json"))) for r in range(world)]
    assert got[0] == got[1] == got[2] == got[3]
    for g, row in enumerate(got[0][:-1]):
        n = 1 + (g % 8)
        assert row == [g + (i % world) + 0.5 for i in range(n)]
    assert got[0][-1] == [9.0]
