"""The C++ proposal core (csrc/search.cpp, ``native.NativeOpEvo``) against
the Python engine and the reference's frozen trajectories.

The core restates numpy's Generator(PCG64) stream (SURVEY.md section 8a RNG
contract) and the reference's ask path (engine.py:132-261, walk.py:41-59,
spaces.py:71-84, 189-221, 266-289, 334-342, 385-387), so every fixture the
Python engine matches must be matched here too.
"""

import json
import os

import numpy as np
import pytest

from paper_2006_05664_b200 import EngineConfig, OpEvo, SearchSpace, make_objective, parse_operator, run
from paper_2006_05664_b200.native import NativeOpEvo, _bind
from paper_2006_05664_b200.spaces import Categorical, Discrete, Factorization, Permutation

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "trajectories.json")) as fh:
    TRAJ = json.load(fh)
with open(os.path.join(HERE, "golden", "replay_hash_objective.json")) as fh:
    REPLAY = json.load(fh)

from test_trajectory_parity import hash_fitness, traj_hash  # noqa: E402


def _core():
    import ctypes as C

    from paper_2006_05664_b200 import capi

    lib = _bind(capi.load())
    h = C.c_void_p()
    assert lib.opevo_search_create(1, (C.c_int32 * 1)(1), (C.c_int64 * 1)(4), None, 8, 8, 0.5, 64,
                                   C.byref(h)) == 0
    return lib, h


@pytest.mark.parametrize("seed", [0, 1, 42, 12345])
def test_pcg64_stream_matches_numpy(seed):
    """random() and integers(n) -- including n = 1 (no draw), the buffered
    32-bit halves surviving intervening random() calls, and the 64-bit path
    -- interleaved exactly as numpy's Generator draws them."""
    import ctypes as C

    lib, h = _core()
    rng = np.random.default_rng(seed)
    s = rng.bit_generator.state
    st, inc = s["state"]["state"], s["state"]["inc"]
    m = (1 << 64) - 1
    lib.opevo_search_set_rng(h, (C.c_uint64 * 4)(st >> 64, st & m, inc >> 64, inc & m), 0, 0)
    draws = np.random.default_rng(seed + 1000)
    ns = [1, 2, 3, 5, 7, 64, 286, 1000, 2 ** 31 - 1, 2 ** 32 - 1, 2 ** 32, 2 ** 32 + 1, 2 ** 40 + 3,
          2 ** 62 + 11]
    out_u, out_d = C.c_uint64(), C.c_double()
    for _ in range(3000):
        if draws.random() < 0.4:
            lib.opevo_search_random(h, C.byref(out_d))
            assert out_d.value == rng.random()
        else:
            n = ns[int(draws.integers(len(ns)))]
            lib.opevo_search_uniform_int(h, n, C.byref(out_u))
            assert out_u.value == int(rng.integers(n))
    lib.opevo_search_destroy(h)


def test_pairwise_sum_matches_numpy():
    import ctypes as C

    lib, h = _core()
    rng = np.random.default_rng(9)
    for n in list(range(1, 300)) + [511, 1024, 1025]:
        a = rng.random(n) * rng.choice([1e-3, 1.0, 1e3], n)
        got = lib.opevo_search_np_sum(a.ctypes.data_as(C.POINTER(C.c_double)), n)
        assert got == float(a.sum()), n
    lib.opevo_search_destroy(h)


@pytest.mark.parametrize("key", sorted(TRAJ["runs"]))
def test_native_synthetic_trajectory_hash(key):
    op, seed = key.split("|")
    space, obj = make_objective(parse_operator(op))
    best, recs = run(space, EngineConfig(seed=int(seed), budget=500), obj, engine_cls=NativeOpEvo)
    want = TRAJ["runs"][key]
    assert len(recs) == want["trials"]
    assert traj_hash(recs) == want["hash"]
    assert best.fitness == want["best_fitness"]


def test_native_mm1_full_sequence():
    space, obj = make_objective(parse_operator("matmul:512,1024,1024"))
    _, recs = run(space, EngineConfig(seed=0, budget=500), obj, engine_cls=NativeOpEvo)
    assert [[r.config, r.fitness] for r in recs] == TRAJ["runs"]["matmul:512,1024,1024|0"]["sequence"]


@pytest.mark.parametrize("seed", sorted(REPLAY["runs"]))
def test_native_replay_all_kinds(seed):
    space = SearchSpace.from_json(REPLAY["space"])
    _, recs = run(space, EngineConfig(seed=int(seed), budget=300),
                  lambda c: hash_fitness(space.config_to_json(c)), engine_cls=NativeOpEvo)
    assert [[r.config, r.fitness] for r in recs] == REPLAY["runs"][seed]["sequence"]


def _lockstep(space, cfg, fitness):
    py, nat = OpEvo(space, cfg), NativeOpEvo(space, cfg)
    gens = 0
    while True:
        a, b = py.ask(), nat.ask()
        assert a.configs == b.configs and a.exhausted == b.exhausted
        if not a.configs:
            break
        fits = [fitness(c) for c in a.configs]
        py.tell(list(zip(a.configs, fits)))
        nat.tell(list(zip(b.configs, fits)))
        gens += 1
        assert py._rng.bit_generator.state == nat.rng_state
    assert py.best().config == nat.best().config
    return gens


@pytest.mark.parametrize("seed", [0, 5])
def test_native_lockstep_with_fallbacks_and_exhaustion(seed):
    """A small space with retry_cap 1 and a budget above its size: the
    native core hands the stream to sample_unvisited (the Python fallback)
    again and again, ties in fitness, zero-fitness generations (uniform
    recombination) and exhaustion all occur."""
    space = SearchSpace([("f", Factorization(12, 2)), ("d", Discrete([1, 2.5, 4])),
                         ("c", Categorical(["a", "b"])), ("p", Permutation(["x", "y", "z"]))])
    cfg = EngineConfig(seed=seed, budget=10_000, parents=3, offspring=5, retry_cap=1,
                       mutation_rate=0.3)
    fit = lambda c: 0.0 if c[2] == "a" else float(c[0][0] % 3)  # noqa: E731 - ties and zeros
    assert _lockstep(space, cfg, fit) > 5


@pytest.mark.parametrize("op", ["conv2d:32,64,56,56,64,3,3,1,1", "batchmatmul:960,128,64,128"])
def test_native_lockstep_operator_spaces(op):
    from paper_2006_05664_b200.mapping import gpu_operator_space

    spec = parse_operator(op)
    space = gpu_operator_space(spec)
    _, obj = make_objective(spec)
    sp0, _ = make_objective(spec)
    # a fitness that depends on every parameter of the B200 space
    fit = lambda c: hash_fitness(space.config_to_json(c))  # noqa: E731
    _lockstep(space, EngineConfig(seed=11, budget=400), fit)
