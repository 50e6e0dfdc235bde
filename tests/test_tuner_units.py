"""Unit tests of the host tuner, modelled on the reference's own suite
(ref pkg/tests/test_spaces.py, test_walk.py, test_engine.py,
test_benchmarks.py), plus known answers frozen from the reference."""

import json
import math
import os
import sys

import numpy as np
import pytest

from paper_2006_05664_b200 import (
    DESK_BATCHMATMUL,
    DESK_CONV2D,
    DESK_MATMUL,
    GOLDEN_OPTIMA,
    Archive,
    Categorical,
    Discrete,
    EngineConfig,
    ExternalEvaluator,
    EvaluatorSpawnError,
    Factorization,
    FatalEvaluationError,
    Individual,
    MatMulSpec,
    OpEvo,
    Permutation,
    ProtocolError,
    SearchSpace,
    build_graph,
    column_sum_deviation,
    enumerate_optimum,
    evaluate_batch,
    is_connected,
    make_objective,
    matmul_space,
    mutate,
    recombine,
    run,
    sample_unvisited,
    sample_walk,
    synthetic_cost,
    walk_distribution,
)
from paper_2006_05664_b200.spaces import parameter_space_from_json

HERE = os.path.dirname(os.path.abspath(__file__))
KA = json.load(open(os.path.join(HERE, "golden", "known_answers.json")))


# ---------------------------------------------------------------- spaces
@pytest.mark.parametrize("case", KA["factorization"], ids=lambda c: f"{c['product']}^{c['arity']}")
def test_factorization_known_answers(case):
    f = Factorization(case["product"], case["arity"])
    assert f.size() == case["size"]
    for idx, val in case["unrank"].items():
        assert list(f.unrank(int(idx))) == val
    for val, nbrs in case["neighbors"].items():
        assert [list(w) for w in f.neighbors(tuple(json.loads(val)))] == nbrs


def test_permutation_known_answers():
    p = Permutation(KA["permutation"]["items"])
    assert [list(p.unrank(i)) for i in range(p.size())] == KA["permutation"]["unrank"]
    assert [list(w) for w in p.neighbors(p.unrank(3))] == KA["permutation"]["neighbors_of_3"]


def test_reference_small_answers():
    # ref pkg/tests/test_spaces.py:79-81, 108-114
    assert Factorization(8, 3).neighbors((8, 1, 1)) == [(4, 1, 2), (4, 2, 1)]
    assert Factorization(8, 3).size() == 10
    assert Factorization(1024, 4).size() == 286
    assert Factorization(4, 2).enumerate() == [(1, 4), (2, 2), (4, 1)]


def test_enumeration_matches_brute_force():
    f = Factorization(72, 3)
    brute = sorted(t for t in __import__("itertools").product(range(1, 73), repeat=3)
                   if math.prod(t) == 72)
    assert f.enumerate() == brute


@pytest.mark.parametrize("space", [Factorization(36, 3), Permutation(("a", "b", "c")),
                                   Discrete((1, 2.5, 7)), Categorical(("x", "y", "z"))])
def test_graphs_connected_and_symmetric(space):
    g = build_graph(space)
    assert is_connected(g)
    for u, adj in enumerate(g.adjacency):
        for w in adj:
            assert u in g.adjacency[w]


def test_invalid_inputs_raise():
    with pytest.raises(ValueError):
        Factorization(0, 2)
    with pytest.raises(ValueError):
        Factorization(8, 3).require((2, 2, 3))
    with pytest.raises(ValueError):
        Discrete((1, 1))
    with pytest.raises(ValueError):
        Categorical(("a", "a"))
    with pytest.raises(ValueError):
        parameter_space_from_json({"kind": "bogus"})
    with pytest.raises(IndexError):
        Factorization(8, 3).unrank(10)


def test_search_space_json_round_trip():
    decl = [{"name": "t", "kind": "factorization", "product": 12, "arity": 3},
            {"name": "o", "kind": "permutation", "items": ["i", "j"]},
            {"name": "u", "kind": "discrete", "values": [0, 16, 64]},
            {"name": "v", "kind": "categorical", "labels": ["on", "off"]}]
    sp = SearchSpace.from_json(decl)
    assert sp.to_json() == decl
    cfg = sp.unrank(17)
    assert sp.config_from_json(json.loads(json.dumps(sp.config_to_json(cfg)))) == cfg
    assert list(sp.iter_configs())[17] == cfg
    with pytest.raises(ValueError):
        sp.config_from_json({"t": [1, 1, 12]})


def test_uniform_sampling_frequencies():
    f = Factorization(12, 2)
    rng = np.random.default_rng(5)
    counts = {}
    for _ in range(30000):
        v = f.sample_uniform(rng)
        counts[v] = counts.get(v, 0) + 1
    assert len(counts) == f.size()
    for c in counts.values():
        assert abs(c / 30000 - 1 / f.size()) < 0.01


def test_sample_unvisited_exhausts():
    sp = SearchSpace([("t", Factorization(8, 2))])
    rng = np.random.default_rng(0)
    seen = set()
    while (c := sample_unvisited(sp, seen, rng, attempts=3)) is not None:
        assert c not in seen
        seen.add(c)
    assert len(seen) == sp.size()


# ------------------------------------------------------------------ walk
@pytest.mark.parametrize("case", KA["walk"], ids=lambda c: c["space"]["kind"])
def test_walk_distribution_known_answers(case):
    sp = parameter_space_from_json(case["space"])
    dist = walk_distribution(build_graph(sp), case["start"], case["rate"])
    np.testing.assert_allclose(dist, case["dist"], atol=1e-12)


def test_walk_hand_solved():
    # ref pkg/tests/test_walk.py:62-70
    np.testing.assert_allclose(walk_distribution(build_graph(Discrete((1, 2, 3))), 0, 0.5),
                               [7 / 12, 1 / 3, 1 / 12], atol=1e-12)
    np.testing.assert_allclose(walk_distribution(build_graph(Discrete((1, 2))), 0, 0.5),
                               [2 / 3, 1 / 3], atol=1e-12)


def test_column_sums_lemma2():
    g = build_graph(Factorization(24, 3))
    assert column_sum_deviation(g, 0.6) < 1e-9


def test_sampler_matches_exact_distribution():
    sp = Factorization(24, 3)
    g = build_graph(sp)
    start = 4
    exact = walk_distribution(g, start, 0.5)
    rng = np.random.default_rng(11)
    emp = np.zeros(len(g))
    draws = 60000
    for _ in range(draws):
        emp[g.index_of(sample_walk(sp, g.vertices[start], 0.5, rng))] += 1
    assert 0.5 * np.abs(emp / draws - exact).sum() < 0.02


def test_rate_zero_never_moves_but_draws():
    rng = np.random.default_rng(1)
    sp = Factorization(64, 3)
    before = rng.bit_generator.state["state"]["state"]
    assert sample_walk(sp, (4, 4, 4), 0.0, rng) == (4, 4, 4)
    assert rng.bit_generator.state["state"]["state"] != before


# ---------------------------------------------------------------- engine
def small_space():
    return SearchSpace([("tile", Factorization(8, 3)), ("flag", Categorical(("on", "off")))])


def index_objective(space):
    ranks = {c: float(i + 1) for i, c in enumerate(space.iter_configs())}
    return lambda c: ranks[c]


def test_engine_config_validation():
    for bad in ({"parents": 0}, {"offspring": 0}, {"mutation_rate": 1.0},
                {"mutation_rate": -0.1}, {"budget": 0}, {"retry_cap": 0}):
        with pytest.raises(ValueError):
            EngineConfig(**bad)


def test_archive_ties_keep_insertion_order():
    a = Archive()
    a.add(Individual(("a",), 2.0))
    a.add(Individual(("b",), 7.0))
    a.add(Individual(("c",), 7.0))
    assert [i.config for i in a.top(3)] == [("b",), ("c",), ("a",)]
    with pytest.raises(ProtocolError):
        a.add(Individual(("a",), 1.0))


def test_recombination_marginals():
    sp = SearchSpace([(f"c{i}", Categorical(("a", "b"))) for i in range(4)])
    parents = [Individual(("a",) * 4, 3.0), Individual(("b",) * 4, 1.0)]
    rng = np.random.default_rng(2024)
    hits = sum(v == "a" for _ in range(50000) for v in recombine(parents, sp, rng))
    assert abs(hits / 200000 - 0.75) < 0.01
    zero = [Individual(("a",) * 4, 5.0), Individual(("b",) * 4, 0.0)]
    assert all(recombine(zero, sp, rng) == ("a",) * 4 for _ in range(2000))


def test_mutation_identity_at_rate_zero():
    sp = small_space()
    rng = np.random.default_rng(0)
    assert mutate(((2, 2, 2), "on"), sp, 0.0, rng) == ((2, 2, 2), "on")


def test_protocol_violations():
    sp = small_space()
    eng = OpEvo(sp, EngineConfig(budget=12, parents=4, offspring=4))
    with pytest.raises(ProtocolError):
        eng.tell([])
    asked = eng.ask()
    with pytest.raises(ProtocolError):
        eng.ask()
    with pytest.raises(ProtocolError):
        eng.tell([(asked.configs[0], 1.0)])
    with pytest.raises(ProtocolError):
        eng.tell([(c, -1.0) for c in asked.configs])
    with pytest.raises(ProtocolError):
        eng.tell([(c, float("nan")) for c in asked.configs])
    eng.tell([(c, 1.0) for c in reversed(asked.configs)])
    assert eng.evaluations == 4


def test_exhaustion_and_no_resample():
    sp = small_space()
    best, recs = run(sp, EngineConfig(budget=500, parents=4, offspring=4, seed=3),
                     index_objective(sp))
    configs = [json.dumps(r.config, sort_keys=True) for r in recs]
    assert len(configs) == len(set(configs)) == sp.size()
    assert best.fitness == float(sp.size())
    eng = OpEvo(sp, EngineConfig(budget=500, parents=4, offspring=4, seed=3))
    while (a := eng.ask()).configs:
        eng.tell([(c, 1.0) for c in a.configs])
    assert eng.ask().exhausted


def test_failures_score_zero_and_fatal_aborts():
    def flaky(c):
        raise RuntimeError("boom")

    assert evaluate_batch(flaky, [1, 2]) == [0.0, 0.0]
    assert evaluate_batch(lambda c: float("inf"), [1]) == [0.0]
    assert evaluate_batch(lambda c: -3, [1]) == [0.0]

    def fatal(c):
        raise FatalEvaluationError("no device")

    with pytest.raises(FatalEvaluationError):
        evaluate_batch(fatal, [1])


def test_evaluate_batch_keeps_order_under_concurrency():
    import time

    def slow(c):
        time.sleep(0.001 * (10 - c))
        return float(c)

    assert evaluate_batch(slow, list(range(10)), concurrency=8) == [float(i) for i in range(10)]


# ------------------------------------------------------------- operators
def test_cost_anchor_and_golden_optima():
    # ref pkg/tests/test_benchmarks.py:115-122 (formula anchor 7/261120) and
    # GOLDEN_OPTIMA via fresh enumeration (ref test_benchmarks.py:193-206)
    for spec in (DESK_MATMUL, DESK_BATCHMATMUL, DESK_CONV2D):
        _, fit = enumerate_optimum(spec)
        assert fit == GOLDEN_OPTIMA[spec.id()]
    spec = MatMulSpec(8, 8, 8)
    sp = matmul_space(spec)
    got = synthetic_cost(spec, sp, ((1, 8, 1, 1), (1, 8, 1, 1), (8, 1, 1)))
    assert math.isclose(got, 7 / 261120, rel_tol=1e-12)
    # threads 1024 is the last valid size; shared overflow scores 0
    assert synthetic_cost(spec, sp, ((1, 1, 8, 1), (1, 1, 8, 1), (1, 1, 8))) > 0.0


def test_external_evaluator_protocol(tmp_path):
    sp = small_space()
    ok = ExternalEvaluator(f"{sys.executable} -c \"import sys,json; "
                           f"d=json.load(sys.stdin); print(len(d['params']['flag']))\"", sp)
    assert ok(((2, 2, 2), "off")) == 3.0
    bad = ExternalEvaluator(f"{sys.executable} -c \"print('nope')\"", sp)
    assert bad(((2, 2, 2), "off")) == 0.0
    slow = ExternalEvaluator(f"{sys.executable} -c \"import time; time.sleep(5)\"", sp,
                             timeout_ms=200)
    assert slow(((2, 2, 2), "off")) == 0.0
    missing = ExternalEvaluator("/nonexistent/evaluator", sp)
    with pytest.raises(EvaluatorSpawnError):
        missing(((2, 2, 2), "off"))


def test_make_objective_default_space():
    sp, obj = make_objective(MatMulSpec(8, 8, 8))
    assert sp.names == ("n", "m", "k")
    assert obj(sp.unrank(0)) >= 0.0
