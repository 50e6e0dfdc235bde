"""Trajectory parity: the host tuner proposes exactly the reference's configs.

Pinned by fixtures frozen from the reference (tests/golden/make_golden.py):
SURVEY.md section 8c hashes for every BASELINE operator x seeds {0, 42},
verbatim first ask batches, the full MM1 sequence, and a replay with a
non-synthetic objective on an extended JSON space (all four parameter kinds).
"""

import hashlib
import json
import os

import pytest

from paper_2006_05664_b200 import (
    EngineConfig,
    OpEvo,
    SearchSpace,
    make_objective,
    parse_operator,
    run,
)

HERE = os.path.dirname(os.path.abspath(__file__))


def _load(name):
    with open(os.path.join(HERE, "golden", name)) as fh:
        return json.load(fh)


TRAJ = _load("trajectories.json")
REPLAY = _load("replay_hash_objective.json")


def traj_hash(records):
    body = "\n".join(json.dumps([r.config, r.fitness]) for r in records)
    return hashlib.sha256(body.encode()).hexdigest()[:16]


def hash_fitness(cfg_json):
    h = hashlib.sha256(json.dumps(cfg_json, sort_keys=True).encode()).digest()
    u = int.from_bytes(h[:8], "little") / 2.0**64
    return 0.0 if u < 0.3 else round(1000.0 * u, 6)


@pytest.mark.parametrize("key", sorted(TRAJ["runs"]))
def test_synthetic_trajectory_hash(key):
    op, seed = key.split("|")
    spec = parse_operator(op)
    space, obj = make_objective(spec)
    best, recs = run(space, EngineConfig(seed=int(seed), budget=500), obj)
    want = TRAJ["runs"][key]
    assert len(recs) == want["trials"]
    assert traj_hash(recs) == want["hash"]
    assert best.fitness == want["best_fitness"]
    assert space.config_to_json(best.config) == want["best_config"]
    assert sum(r.fitness == 0.0 for r in recs) == want["zeros"]


@pytest.mark.parametrize("key", sorted(TRAJ["runs"]))
def test_first_two_asks_verbatim(key):
    op, seed = key.split("|")
    space, obj = make_objective(parse_operator(op))
    eng = OpEvo(space, EngineConfig(seed=int(seed), budget=500))
    for want in TRAJ["runs"][key]["first_asks"]:
        got = eng.ask()
        assert [space.config_to_json(c) for c in got.configs] == want
        eng.tell([(c, obj(c)) for c in got.configs])


def test_mm1_full_sequence():
    space, obj = make_objective(parse_operator("matmul:512,1024,1024"))
    _, recs = run(space, EngineConfig(seed=0, budget=500), obj)
    want = TRAJ["runs"]["matmul:512,1024,1024|0"]["sequence"]
    got = [[r.config, r.fitness] for r in recs]
    assert got == want


@pytest.mark.parametrize("seed", sorted(REPLAY["runs"]))
def test_replayed_arbitrary_objective_all_kinds(seed):
    space = SearchSpace.from_json(REPLAY["space"])
    _, recs = run(space, EngineConfig(seed=int(seed), budget=300),
                  lambda c: hash_fitness(space.config_to_json(c)))
    want = REPLAY["runs"][seed]
    assert [[r.config, r.fitness] for r in recs] == want["sequence"]
    assert traj_hash(recs) == want["hash"]


def test_lockstep_against_live_reference(reference_topotune):
    """Reference OpEvo and ours receive identical fitness; every ask must match."""
    tt = reference_topotune
    space_json = REPLAY["space"]
    ref_space = tt.SearchSpace.from_json(space_json)
    our_space = SearchSpace.from_json(space_json)
    for seed in (3, 7):
        ref = tt.OpEvo(ref_space, tt.EngineConfig(seed=seed, budget=200, parents=4, offspring=6,
                                                  mutation_rate=0.7))
        ours = OpEvo(our_space, EngineConfig(seed=seed, budget=200, parents=4, offspring=6,
                                             mutation_rate=0.7))
        while True:
            a, b = ref.ask(), ours.ask()
            assert a.configs == b.configs and a.exhausted == b.exhausted
            if not a.configs:
                break
            fits = [hash_fitness(our_space.config_to_json(c)) for c in a.configs]
            ref.tell(list(zip(a.configs, fits)))
            ours.tell(list(zip(b.configs, fits)))
        assert ref.best().config == ours.best().config
