"""``NativeOpEvo``: OpEvo whose proposals come from the C++ search core.

Same class contract as :class:`engine.OpEvo` (ask / tell / best, the
``archive``, ``EngineConfig``, ``ProtocolError``), same proposals bit for bit
under the same told fitness -- the reference's ask path
(``pkg/src/topotune/engine.py:181-261``) restated in ``csrc/search.cpp`` over
numpy's PCG64 stream.  What stays in Python: the budget / exhaustion checks
of ``ask`` (engine.py:181-197), ``tell``'s validation, and the rare
``sample_unvisited`` fallback (spaces.py:614-647), for which the generator
state is handed to numpy and back.

Why: the Python ask costs ~0.2 ms per generation -- a third of a generation
once trials are sharded one per GPU; the native core
takes a few microseconds.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import capi
from .engine import AskResult, EngineConfig, OpEvo, ProtocolError
from .spaces import Categorical, Discrete, Factorization, Permutation, SearchSpace, sample_unvisited

_KIND = {Factorization: 0, Discrete: 1, Categorical: 2, Permutation: 3}
_U64_MASK = (1 << 64) - 1


def _bind(lib):
    if getattr(lib, "_search_bound", False):
        return lib
    P, I, D = C.c_void_p, C.c_int, C.c_double
    i64p, u64p = C.POINTER(C.c_int64), C.POINTER(C.c_uint64)
    sig = {
        "opevo_search_create": (I, [I, C.POINTER(C.c_int32), i64p, C.POINTER(C.c_int32), I, I, D, I,
                                    C.POINTER(P)]),
        "opevo_search_destroy": (None, [P]),
        "opevo_search_slots": (I, [P]),
        "opevo_search_set_rng": (I, [P, u64p, I, C.c_uint32]),
        "opevo_search_get_rng": (I, [P, u64p, C.POINTER(I), C.POINTER(C.c_uint32)]),
        "opevo_search_propose": (I, [P, I, I, I, i64p, C.POINTER(I)]),
        "opevo_search_add_pending": (I, [P, i64p]),
        "opevo_search_tell": (I, [P, I, i64p, C.POINTER(C.c_double)]),
        "opevo_search_uniform_int": (I, [P, C.c_uint64, u64p]),
        "opevo_search_random": (I, [P, C.POINTER(C.c_double)]),
        "opevo_search_np_sum": (D, [C.POINTER(C.c_double), C.c_size_t]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    lib._search_bound = True
    return lib


def native_supported(space: SearchSpace) -> bool:
    """Every parameter kind is served natively except permutations of more
    than 20 items (their uniform draw exceeds 2^63 and uses byte rejection)."""
    for s in space.spaces:
        if type(s) not in _KIND:
            return False
        if isinstance(s, Permutation) and len(s.items) > 20:
            return False
    return True


class _Codec:
    """Configuration tuples <-> int64 slot rows (see include/opevo.h)."""

    def __init__(self, space: SearchSpace):
        self.space = space
        self.kinds, self.a, self.arity = [], [], []
        self.dec, self.enc = [], []
        for s in space.spaces:
            k = _KIND[type(s)]
            self.kinds.append(k)
            if isinstance(s, Factorization):
                self.a.append(s.product)
                self.arity.append(s.arity)
                self.dec.append((s.arity, tuple))
                self.enc.append(lambda v: v)
            elif isinstance(s, Permutation):
                items = s.items
                rank = {x: i for i, x in enumerate(items)}
                self.a.append(len(items))
                self.arity.append(len(items))
                self.dec.append((len(items), lambda row, items=items: tuple(items[j] for j in row)))
                self.enc.append(lambda v, rank=rank: tuple(rank[x] for x in v))
            elif isinstance(s, Discrete):
                vals = s.values
                pos = s._pos
                self.a.append(len(vals))
                self.arity.append(1)
                self.dec.append((1, lambda row, vals=vals: vals[row[0]]))
                self.enc.append(lambda v, pos=pos: (pos[v],))
            else:
                labels = s.labels
                pos = {x: i for i, x in enumerate(labels)}
                self.a.append(len(labels))
                self.arity.append(1)
                self.dec.append((1, lambda row, labels=labels: labels[row[0]]))
                self.enc.append(lambda v, pos=pos: (pos[v],))
        self.slots = sum(self.arity)

    def decode(self, row) -> tuple:
        out, o = [], 0
        for n, f in self.dec:
            out.append(f(row[o:o + n]))
            o += n
        return tuple(out)

    def encode(self, config: tuple) -> list[int]:
        row: list[int] = []
        for f, v in zip(self.enc, config):
            row.extend(f(v))
        return row


class NativeOpEvo(OpEvo):
    """:class:`engine.OpEvo` with the proposal loop in ``libopevo``."""

    def __init__(self, space: SearchSpace, config: EngineConfig | None = None) -> None:
        super().__init__(space, config)
        if not native_supported(space):
            raise ValueError("space has a parameter the native core does not serve")
        self._lib = _bind(capi.load())
        self._codec = _Codec(space)
        cfg = self.config
        n = len(space.spaces)
        h = C.c_void_p()
        st = self._lib.opevo_search_create(
            n, (C.c_int32 * n)(*self._codec.kinds), (C.c_int64 * n)(*self._codec.a),
            (C.c_int32 * n)(*self._codec.arity), cfg.parents, cfg.offspring, float(cfg.mutation_rate),
            cfg.retry_cap, C.byref(h))
        if st != capi.OK:
            raise ValueError(f"native search core rejected the space/config (status {st})")
        self._h = h
        self._slots = self._codec.slots
        self._push_rng()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._lib.opevo_search_destroy(h)
            self._h = None

    # -- RNG hand-over (numpy PCG64 state <-> the native stream) -------------
    def _push_rng(self) -> None:
        s = self._rng.bit_generator.state
        st, inc = s["state"]["state"], s["state"]["inc"]
        arr = (C.c_uint64 * 4)(st >> 64, st & _U64_MASK, inc >> 64, inc & _U64_MASK)
        self._lib.opevo_search_set_rng(self._h, arr, int(s["has_uint32"]), int(s["uinteger"]))

    def _pull_rng(self) -> None:
        arr = (C.c_uint64 * 4)()
        has, u = C.c_int(), C.c_uint32()
        self._lib.opevo_search_get_rng(self._h, arr, C.byref(has), C.byref(u))
        self._rng.bit_generator.state = {
            "bit_generator": "PCG64",
            "state": {"state": (arr[0] << 64) | arr[1], "inc": (arr[2] << 64) | arr[3]},
            "has_uint32": has.value, "uinteger": u.value}

    # -- proposals ------------------------------------------------------------
    def _native_batch(self, want: int, initial: bool) -> list[tuple]:
        out = (C.c_int64 * (max(want, 1) * self._slots))()
        need = C.c_int()
        batch: list[tuple] = []
        rows: list[int] = []
        first = 1
        while len(batch) < want:
            left = want - len(batch)
            made = self._lib.opevo_search_propose(self._h, int(initial), first, left, out, C.byref(need))
            first = 0
            if made < 0:
                raise RuntimeError(f"native search core failed (status {made})")
            flat = out[:made * self._slots]
            rows.extend(flat)
            for i in range(made):
                batch.append(self._codec.decode(flat[i * self._slots:(i + 1) * self._slots]))
            if need.value:
                # retry cap exhausted: the reference's sample_unvisited, drawn
                # from the same stream (engine.py:240-241, 257-258)
                self._pull_rng()
                visited = set(batch) if initial else self.archive.configs() | set(batch)
                pick = sample_unvisited(self.space, visited, self._rng)
                self._push_rng()
                row = self._codec.encode(pick)
                self._lib.opevo_search_add_pending(self._h, (C.c_int64 * self._slots)(*row))
                rows.extend(row)
                batch.append(pick)
        self._rows = rows           # slot form of the batch, for tell()
        return batch

    def _initial_batch(self, want: int) -> list[tuple]:
        return self._native_batch(want, True)

    def _offspring_batch(self, want: int) -> list[tuple]:
        return self._native_batch(want, False)

    def tell(self, results) -> None:
        pending = self._pending
        super().tell(results)                 # validation + the Python archive
        # the native archive, in ask order with the told fitness
        got = {}
        for cfg, fit in results:
            got[tuple(cfg)] = float(fit)
        rows = self._rows
        n = len(pending)
        st = self._lib.opevo_search_tell(self._h, n, (C.c_int64 * len(rows))(*rows),
                                         (C.c_double * n)(*[got[c] for c in pending]))
        if st != capi.OK:
            raise ProtocolError(f"native archive rejected the batch (status {st})")

    @property
    def rng_state(self) -> dict:
        """numpy's view of the stream after the last proposal."""
        self._pull_rng()
        return self._rng.bit_generator.state


def make_engine(space: SearchSpace, config: EngineConfig | None = None, native: bool = True) -> OpEvo:
    """The native engine when the library is built and the space is served,
    else the Python one (identical proposals either way)."""
    if native and native_supported(space):
        try:
            return NativeOpEvo(space, config)
        except OSError:
            pass
    return OpEvo(space, config)
