"""Random search / simulated annealing / G-BFS reproduce the reference's
seeded trajectories (fixtures frozen from the reference, tests/golden)."""

import hashlib
import json
import os

import pytest

from paper_2006_05664_b200 import make_objective, parse_operator
from paper_2006_05664_b200.baselines import (
    GbfsConfig,
    SaConfig,
    calibrate_temperature,
    greedy_bfs,
    metropolis_accept,
    random_search,
    simulated_annealing,
)

HERE = os.path.dirname(os.path.abspath(__file__))
BASE = json.load(open(os.path.join(HERE, "golden", "baselines.json")))


def traj_hash(records):
    body = "\n".join(json.dumps([r.config, r.fitness]) for r in records)
    return hashlib.sha256(body.encode()).hexdigest()[:16]


@pytest.mark.parametrize("key", sorted(BASE["runs"]))
def test_baseline_trajectory_matches_reference(key):
    op, name, seed = key.split("|")
    space, obj = make_objective(parse_operator(op))
    seed = int(seed)
    if name == "random":
        best, recs = random_search(space, 300, seed, obj)
    elif name == "sa":
        best, recs = simulated_annealing(space, SaConfig(), 300, seed, obj)
    else:
        best, recs = greedy_bfs(space, GbfsConfig(), 300, seed, obj)
    want = BASE["runs"][key]
    assert len(recs) == want["trials"]
    assert best.fitness == want["best"]
    assert traj_hash(recs) == want["hash"]


def test_config_validation_and_helpers():
    import numpy as np

    with pytest.raises(ValueError):
        SaConfig(cooling=1.0)
    with pytest.raises(ValueError):
        GbfsConfig(pool_size=0)
    assert calibrate_temperature([1.0, 1.0]) == 1.0
    rng = np.random.default_rng(0)
    assert metropolis_accept(rng, 1.0, 2.0, 0.5)
    assert not metropolis_accept(rng, 2.0, 1.0, 0.0)


def test_cli_compare_synthetic(tmp_path):
    from paper_2006_05664_b200.__main__ import main

    assert main(["compare", "--operator", "matmul:16,16,16", "--evaluator", "synthetic",
                 "--budget", "40", "--seeds", "0,1", "--out", str(tmp_path)]) == 0
    assert (tmp_path / "summary.csv").exists() and (tmp_path / "curves.csv").exists()
    assert main(["tune", "--operator", "matmul:16,16,16", "--evaluator", "synthetic",
                 "--budget", "20", "--out", str(tmp_path)]) == 0


def test_cli_gpu_unavailable_exit_code(tmp_path):
    if os.path.exists("/dev/nvidia0"):
        pytest.skip("a GPU is present")
    from paper_2006_05664_b200.__main__ import main

    assert main(["tune", "--operator", "matmul:256,256,256", "--budget", "8",
                 "--out", str(tmp_path)]) == 3
