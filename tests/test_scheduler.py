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
from paper_2006_05664_b200.evaluator import TrialInfo
from paper_2006_05664_b200.mapping import config_to_knobs, gpu_operator_space
from paper_2006_05664_b200.scheduler import ShardedEvaluator, shard_indices

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


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    space = gpu_operator_space(SPEC)
    ev = ShardedEvaluator(None, rank, world, local_fn=fake_infos(space, rank))
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


def test_two_rank_gloo_sharding_matches_single_process():
    space = gpu_operator_space(SPEC)
    # single-process reference trajectory with the same fitness function
    local = fake_infos(space, 0)
    _, single = run(space, EngineConfig(seed=5, budget=96), lambda c: local([c])[0].fitness)
    with tempfile.TemporaryDirectory() as d:
        tmp.start_processes(_worker, args=(2, _free_port(), d), nprocs=2, start_method="spawn")
        r0 = json.load(open(os.path.join(d, "r0.json")))
        r1 = json.load(open(os.path.join(d, "r1.json")))
    want = [[r.config, r.fitness] for r in single]
    assert r0["seq"] == r1["seq"] == want
    # ask index i was evaluated by rank i % 2 within every generation of 8
    assert r0["gpus"][:8] == [0, 1] * 4
