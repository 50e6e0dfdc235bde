"""Compact restatement of the reference tuner -- TEST INFRASTRUCTURE ONLY.

The reference (``topotune`` 0.1.0, ``/root/reference/pkg/src/topotune``) is pure
Python + numpy; this port restates its OpEvo loop and its CPU evaluator (the
synthetic cost model) in one file, independently of the product package, so
that

* ``bench.py --impl reference`` / ``cpu_baseline`` can time "the reference's
  own CPU implementation of the path" on the GPU box (the reference tree is
  not present there);
* the tests can cross-check the product tuner against a second
  implementation.

Pinned by tests/golden/trajectories.json (hashes frozen from the reference
itself): tests/test_oracle_port.py asserts bit-identical trajectories.

Third-party arithmetic: numpy's ``Generator(PCG64)`` (unpinned ``numpy>=1.24``
in ``pkg/pyproject.toml:11``; fixtures frozen with numpy 2.3.5) is used
directly, as the reference does.
"""

from __future__ import annotations

import bisect
import math

import numpy as np


# ---------------------------------------------------------------- spaces
# ref spaces.py:36-84
def _pfact(n):
    f, d = {}, 2
    while d * d <= n:
        while n % d == 0:
            f[d] = f.get(d, 0) + 1
            n //= d
        d += 1 if d == 2 else 2
    if n > 1:
        f[n] = f.get(n, 0) + 1
    return f


def _count(f, slots):
    c = 1
    for e in f.values():
        c *= math.comb(e + slots - 1, slots - 1)
    return c


def _divs(f):
    ds = [1]
    for p, e in f.items():
        ds = [d * p ** k for d in ds for k in range(e + 1)]
    return sorted(ds)


def _uniform(rng, n):
    if n <= (1 << 63) - 1:
        return int(rng.integers(n))
    bits = n.bit_length()
    while True:
        r = int.from_bytes(rng.bytes((bits + 7) // 8), "big") & ((1 << bits) - 1)
        if r < n:
            return r


class Fact:
    """Factorization parameter (ref spaces.py:140-231)."""

    def __init__(self, product, arity):
        self.product, self.arity = product, arity
        self.f = _pfact(product)
        self.primes = sorted(self.f)
        self.n = _count(self.f, arity)

    def unrank(self, i):
        out, rem = [], self.product
        for slots in range(self.arity - 1, 0, -1):
            for d in _divs(_pfact(rem)):
                c = _count(_pfact(rem // d), slots)
                if i < c:
                    out.append(d)
                    rem //= d
                    break
                i -= c
        return tuple(out + [rem])

    def neighbors(self, v):
        s = set()
        for a in range(self.arity):
            for p in self.primes:
                if v[a] % p == 0:
                    for b in range(self.arity):
                        if b != a:
                            w = list(v)
                            w[a] //= p
                            w[b] *= p
                            s.add(tuple(w))
        return sorted(s)


class Disc:
    """Discrete path parameter (ref spaces.py:303-356)."""

    def __init__(self, values):
        self.values = tuple(values)
        self.n = len(self.values)

    def unrank(self, i):
        return self.values[i]

    def neighbors(self, v):
        i = self.values.index(v)
        return [self.values[j] for j in (i - 1, i + 1) if 0 <= j < self.n]


class Cat:
    """Categorical complete-graph parameter (ref spaces.py:359-400)."""

    def __init__(self, labels):
        self.labels = tuple(labels)
        self.n = len(self.labels)

    def unrank(self, i):
        return self.labels[i]

    def neighbors(self, v):
        return [x for x in self.labels if x != v]


def operator_params(op: str):
    """(names, params, spec tuple) of a reference operator string
    (ref benchmarks.py:113-175)."""
    kind, _, dims = op.partition(":")
    d = [int(x) for x in dims.split(",")]
    if kind == "matmul":
        n, m, k = d
        return ("n", "m", "k"), [Fact(n, 4), Fact(m, 4), Fact(k, 3)], ("mm", d)
    if kind == "batchmatmul":
        b, n, m, k = d
        return ("b", "n", "m", "k"), [Fact(b, 2), Fact(n, 4), Fact(m, 4), Fact(k, 3)], ("bmm", d)
    if kind == "conv2d":
        B, ci, h, w, co, kh, kw, s, p = d
        ho, wo = (h + 2 * p - kh) // s + 1, (w + 2 * p - kw) // s + 1
        return (("co", "ho", "wo", "ci", "kh", "kw", "unroll_explicit", "unroll_step"),
                [Fact(co, 4), Fact(ho, 4), Fact(wo, 4), Fact(ci, 2), Fact(kh, 2), Fact(kw, 2),
                 Cat(("explicit_unroll_on", "explicit_unroll_off")),
                 Disc((0, 16, 64, 512, 1500))], ("conv", d))
    raise ValueError(op)


# ------------------------------------------------------- synthetic evaluator
# ref benchmarks.py:211-291 (DEFAULT_COST_PARAMS)
def synthetic_cost(kind, names, cfg):
    v = dict(zip(names, cfg))
    if kind in ("mm", "bmm"):
        n, m, k = v["n"], v["m"], v["k"]
        threads, shared = n[2] * m[2], (n[2] * n[3] + m[2] * m[3]) * k[2]
        reg, grid, inner, bonus = n[3] * m[3], n[0] * m[0], k[2], 1.0
        if kind == "bmm":
            grid *= v["b"][0]
    else:
        co, ho, wo, ci, kh, kw = (v[x] for x in ("co", "ho", "wo", "ci", "kh", "kw"))
        threads = co[2] * ho[2] * wo[2]
        shared = (co[2] * co[3] + ci[1]) * kh[1] * kw[1] * 8
        reg, grid, inner = co[3] * ho[3] * wo[3], co[0] * ho[0] * wo[0], kh[1] * kw[1]
        bonus = 1.05 if (v["unroll_explicit"] == "explicit_unroll_on" and v["unroll_step"] >= 64) else 1.0
    if threads > 1024 or shared > 12288:
        return 0.0
    occ = (min(threads, 256) / 256) * math.sqrt(256 / max(threads, 256))
    return 10.0 * occ * (reg / (reg + 16.0)) * (1.0 if inner in (4, 8, 16) else 0.7) * \
        (min(grid, 60) / 60) * bonus


# ---------------------------------------------------------------- OpEvo
def _walk(p, v, q, rng):                                   # ref walk.py:41-59
    for _ in range(1_000_000):
        if rng.random() >= q:
            return v
        nb = p.neighbors(v)
        if not nb:
            return v
        v = nb[int(rng.integers(len(nb)))]
    raise RuntimeError("walk did not stop")


def _unvisited(params, visited, rng):                      # ref spaces.py:614-647
    total = math.prod(p.n for p in params)
    if total - len(visited) <= 0:
        return None
    for _ in range(1000):
        c = tuple(p.unrank(_uniform(rng, p.n)) for p in params)
        if c not in visited:
            return c
    raise RuntimeError("rejection sampling exhausted (enumeration path not restated)")


def opevo_run(op: str, seed: int = 0, budget: int = 500, lam: int = 8, rho: int = 8,
              q: float = 0.5, retry_cap: int = 64, objective=None):
    """Reference ``run(space, EngineConfig(...), objective)`` (engine.py:293-310).
    Returns the list of (config, fitness) in trial order."""
    names, params, (kind, _) = operator_params(op)
    obj = objective or (lambda c: synthetic_cost(kind, names, c))
    rng = np.random.default_rng(seed)
    keys, ranked, seen = [], [], set()
    log = []
    total = math.prod(p.n for p in params)
    while True:
        done = len(log)
        if total - done <= 0 or budget - done <= 0:
            break
        batch, taken = [], set()
        if done == 0:                                      # ref engine.py:228-242
            for _ in range(min(lam, budget, total)):
                pick = None
                for _ in range(retry_cap):
                    c = tuple(p.unrank(_uniform(rng, p.n)) for p in params)
                    if c not in taken:
                        pick = c
                        break
                pick = pick or _unvisited(params, taken, rng)
                batch.append(pick)
                taken.add(pick)
        else:                                              # ref engine.py:244-261
            parents = ranked[:lam]
            fit = np.array([f for _, f in parents], dtype=float)
            tot = fit.sum()
            for _ in range(min(rho, budget - done, total - done)):
                picks = rng.choice(len(parents), size=len(params),
                                   p=fit / tot if tot > 0.0 else None)
                base = tuple(parents[int(j)][0][i] for i, j in enumerate(picks))
                pick = None
                for _ in range(retry_cap):
                    c = tuple(_walk(p, v, q, rng) for p, v in zip(params, base))
                    if c not in seen and c not in taken:
                        pick = c
                        break
                pick = pick or _unvisited(params, seen | taken, rng)
                batch.append(pick)
                taken.add(pick)
        fits = []
        for c in batch:                                    # ref engine.py:276-285
            try:
                f = float(obj(c))
            except Exception:   # noqa: BLE001
                f = 0.0
            fits.append(f if math.isfinite(f) and f >= 0.0 else 0.0)
        for c, f in zip(batch, fits):                      # tell, ask order
            i = bisect.bisect_right(keys, -f)
            keys.insert(i, -f)
            ranked.insert(i, (c, f))
            seen.add(c)
            log.append((c, f))
    return names, log
