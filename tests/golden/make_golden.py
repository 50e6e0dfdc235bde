"""Freeze golden vectors from the reference tuner (run in the build container).

The reference (``/root/reference/pkg/src/topotune``, pure Python + numpy) is
imported read-only and run on the BASELINE configurations; its outputs are
written as small JSON fixtures next to this script.  The GPU box has no
``/root/reference``, so the tests compare against these files.

Fixtures:
* ``trajectories.json`` -- for every BASELINE operator x seeds {0, 42}:
  sha256 of the (config, fitness) sequence of ``run(space,
  EngineConfig(seed, budget=500), synthetic objective)`` (the SURVEY.md
  section 8c hash definition), the best fitness, the zero count and the
  first two ask batches verbatim.  For MM1 the full 500-trial sequence is kept.
* ``replay_hash_objective.json`` -- the same loop with a non-synthetic
  objective (a config hash with a 30 % invalid region) on the B200 GPU space,
  to pin trajectory parity under arbitrary replayed fitness values.
* ``known_answers.json`` -- unrank / neighbours / sizes / exact walk laws.

Usage: ``python tests/golden/make_golden.py`` (numpy version recorded).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OPERATORS = [
    "matmul:512,1024,1024",
    "matmul:1024,1024,1024",
    "batchmatmul:960,128,64,128",
    "conv2d:32,64,56,56,64,3,3,1,1",
    "matmul:4096,4096,4096",
]
SEEDS = [0, 42]


def traj_hash(records) -> str:
    body = "\n".join(json.dumps([r.config, r.fitness]) for r in records)
    return hashlib.sha256(body.encode()).hexdigest()[:16]


def hash_fitness(cfg_json: dict) -> float:
    """Deterministic non-synthetic fitness: 0 for ~30 % of configs."""
    h = hashlib.sha256(json.dumps(cfg_json, sort_keys=True).encode()).digest()
    u = int.from_bytes(h[:8], "little") / 2.0**64
    return 0.0 if u < 0.3 else round(1000.0 * u, 6)


def main() -> None:
    sys.path.insert(0, REF_SRC)
    import topotune as tt
    from topotune import spaces as tsp
    from topotune.walk import walk_distribution

    out = {"numpy": np.__version__, "reference": "topotune " + tt.__version__, "runs": {}}
    for op in OPERATORS:
        spec = tt.parse_operator(op)
        space, obj = tt.make_objective(spec)
        for seed in SEEDS:
            eng = tt.OpEvo(space, tt.EngineConfig(seed=seed, budget=500))
            asks = []
            for _ in range(2):
                a = eng.ask()
                asks.append([space.config_to_json(c) for c in a.configs])
                eng.tell([(c, obj(c)) for c in a.configs])
            best, recs = tt.run(space, tt.EngineConfig(seed=seed, budget=500), obj)
            entry = {
                "hash": traj_hash(recs),
                "trials": len(recs),
                "best_fitness": best.fitness,
                "best_config": space.config_to_json(best.config),
                "zeros": sum(1 for r in recs if r.fitness == 0.0),
                "first_asks": asks,
            }
            if op == "matmul:512,1024,1024":
                entry["sequence"] = [[r.config, r.fitness] for r in recs]
            out["runs"][f"{op}|{seed}"] = entry
    with open(os.path.join(HERE, "trajectories.json"), "w") as fh:
        json.dump(out, fh, separators=(",", ":"))

    # replay with an arbitrary objective on an extended (GPU-style) JSON space
    space_json = [
        {"name": "n", "kind": "factorization", "product": 1024, "arity": 4},
        {"name": "m", "kind": "factorization", "product": 1024, "arity": 4},
        {"name": "k", "kind": "factorization", "product": 1024, "arity": 3},
        {"name": "stages", "kind": "discrete", "values": [2, 3, 4, 5, 6, 7, 8]},
        {"name": "raster", "kind": "categorical", "labels": ["row", "col"]},
        {"name": "order", "kind": "permutation", "items": ["i", "j", "k"]},
    ]
    space = tt.SearchSpace.from_json(space_json)
    replay = {"numpy": np.__version__, "space": space_json, "runs": {}}
    for seed in SEEDS:
        best, recs = tt.run(space, tt.EngineConfig(seed=seed, budget=300),
                            lambda c: hash_fitness(space.config_to_json(c)))
        replay["runs"][str(seed)] = {
            "hash": traj_hash(recs),
            "sequence": [[r.config, r.fitness] for r in recs],
        }
    with open(os.path.join(HERE, "replay_hash_objective.json"), "w") as fh:
        json.dump(replay, fh, separators=(",", ":"))

    # baselines (ref baselines.py) on MM1 and the desk conv, synthetic objective
    base = {"numpy": np.__version__, "runs": {}}
    for op in ("matmul:512,1024,1024", "conv2d:1,4,8,8,8,3,3,1,1"):
        spec = tt.parse_operator(op)
        space, obj = tt.make_objective(spec)
        for seed in SEEDS:
            for name, fn in (("random", lambda: tt.random_search(space, 300, seed, obj)),
                             ("sa", lambda: tt.simulated_annealing(space, tt.SaConfig(), 300, seed, obj)),
                             ("gbfs", lambda: tt.greedy_bfs(space, tt.GbfsConfig(), 300, seed, obj))):
                best, recs = fn()
                base["runs"][f"{op}|{name}|{seed}"] = {"hash": traj_hash(recs), "trials": len(recs),
                                                        "best": best.fitness}
    with open(os.path.join(HERE, "baselines.json"), "w") as fh:
        json.dump(base, fh, indent=1)

    # known answers: unrank, neighbours, sizes, walk laws
    ka: dict = {"factorization": [], "permutation": [], "walk": []}
    for prod, arity in [(8, 3), (1024, 4), (1024, 3), (960, 2), (56, 4), (720, 3), (64, 4)]:
        f = tsp.Factorization(prod, arity)
        n = f.size()
        idx = sorted({0, 1, n // 3, n // 2, n - 1})
        vals = [list(f.unrank(i)) for i in idx]
        nb = {json.dumps(v): [list(w) for w in f.neighbors(tuple(v))] for v in vals}
        ka["factorization"].append({"product": prod, "arity": arity, "size": n,
                                    "unrank": dict(zip(map(str, idx), vals)),
                                    "neighbors": nb})
    p = tsp.Permutation(("i", "j", "k", "l"))
    ka["permutation"] = {"items": list(p.items),
                         "unrank": [list(p.unrank(i)) for i in range(p.size())],
                         "neighbors_of_3": [list(w) for w in p.neighbors(p.unrank(3))]}
    for space_j, start, rate in [({"kind": "discrete", "values": [1, 2, 3]}, 0, 0.5),
                                 ({"kind": "factorization", "product": 12, "arity": 2}, 1, 0.5),
                                 ({"kind": "categorical", "labels": ["a", "b", "c"]}, 2, 0.3)]:
        sp = tsp.parameter_space_from_json(space_j)
        dist = walk_distribution(tsp.build_graph(sp), start, rate)
        ka["walk"].append({"space": space_j, "start": start, "rate": rate,
                           "dist": [float(x) for x in dist]})
    with open(os.path.join(HERE, "known_answers.json"), "w") as fh:
        json.dump(ka, fh, indent=1)
    print("golden fixtures written with numpy", np.__version__)


if __name__ == "__main__":
    main()
