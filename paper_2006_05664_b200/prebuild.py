"""Ahead-of-time population of the cubin cache (host NVRTC pool, no GPU).

Enumerates the distinct kernel instances that an operator's GPU search space
can map to (``mapping.config_to_knobs``) and compiles each once into
``kernel_cache/``.  A tuning run then pays only module loads; bench.py
reports cache hits and the compile time a cold cache would have cost.
"""

from __future__ import annotations

import itertools
import os
import time
from concurrent.futures import ThreadPoolExecutor

from . import capi
from .mapping import (
    FAMILY_TF32X3,
    STAGE_VALUES,
    UNROLL_TO_STAGES,
    Knobs,
    _bk_ok,
    _conv_resident_fit,
    _fit_halo_stages,
    _fit_stages,
)
from .operators import BatchMatMulSpec, Conv2dSpec, MatMulSpec, parse_operator


def _divisors(n: int) -> list[int]:
    return [d for d in range(1, n + 1) if n % d == 0]


def _x3_instances(spec) -> set[tuple[int, bool, tuple]]:
    """3xTF32 family (fp32 MatMul / BMM on tcgen05): mirrors mapping._x3_knobs."""
    out = set()
    batched = isinstance(spec, BatchMatMulSpec)
    for bm in (128, 256):
        if spec.n % bm:
            continue
        for bn in range(16, 257, 16):
            if spec.m % bn or (2 if bm == 256 else 1) * bn > 512:
                continue
            for bk in _divisors(spec.k):
                if not _bk_ok(2 * bk):
                    continue
                for st in STAGE_VALUES:
                    s = _fit_stages(st, bm, bn, bk, x3=True)
                    if s < 1:
                        continue
                    out.add((FAMILY_TF32X3, batched, Knobs(bm, bn, bk, s, family=FAMILY_TF32X3).as_tuple()))
                    if bm == 128:
                        for sp in (2, 4, 8):
                            kn = Knobs(bm, bn, bk, s, sp, family=FAMILY_TF32X3, batched=int(batched))
                            if kn.dsmem_split() and spec.k % (sp * bk) == 0:
                                out.add((FAMILY_TF32X3, batched, kn.as_tuple()))
    return out


def _representatives(space, key) -> list:
    """One value per distinct key(value) of a parameter space."""
    seen = {}
    for v in space.enumerate():
        seen.setdefault(key(v), v)
    return list(seen.values())


def _conv_instances(spec) -> set[tuple[int, bool, tuple]]:
    """Conv instances reachable from conv2d_space: the mapping itself
    (mapping._conv_knobs) over one representative configuration per
    combination of the parameter features it reads -- co[0], co[1] mod 4,
    ho[0], ho[1] parity, wo[0], ci[0], kh[0] * kw[0], unroll settings."""
    from .mapping import _conv_knobs
    from .operators import conv2d_space

    space = conv2d_space(spec)
    sp = dict(zip(space.names, space.spaces))
    reps = {
        "co": _representatives(sp["co"], lambda v: (v[0], v[1] % 4)),
        "ho": _representatives(sp["ho"], lambda v: (v[0], v[1] % 2)),
        "wo": _representatives(sp["wo"], lambda v: v[0]),
        "ci": _representatives(sp["ci"], lambda v: v[0]),
        "kh": _representatives(sp["kh"], lambda v: v[0]),
        "kw": _representatives(sp["kw"], lambda v: v[0]),
        "unroll_explicit": list(sp["unroll_explicit"].labels),
        "unroll_step": list(sp["unroll_step"].values),
    }
    out = set()
    for combo in itertools.product(*(reps[n] for n in space.names)):
        kn, _ = _conv_knobs(spec, dict(zip(space.names, combo)))
        if kn is not None:
            out.add((1, False, kn.as_tuple()))
    return out


def family_instances(spec, dtype: str = "bf16") -> set[tuple[int, bool, tuple]]:
    """All (family, batched, knobs) reachable from the operator's space."""
    out = set()
    if dtype == "tf32x3":
        return _x3_instances(spec)
    if isinstance(spec, (MatMulSpec, BatchMatMulSpec)):
        batched = isinstance(spec, BatchMatMulSpec)
        for bm in (128, 256):
            if spec.n % bm:
                continue
            for bn in range(16, 257, 16):
                if spec.m % bn:
                    continue
                grid_cols = spec.m // bn
                clusters = {c for c in (1, 2, 4) if grid_cols % c == 0}
                for bk in _divisors(spec.k):
                    if not _bk_ok(bk):
                        continue
                    for cg in ((1, 2) if bm == 256 else (1,)):
                        if cg == 1 and bm == 256 and bn > 256:
                            continue
                        for st in STAGE_VALUES:
                            s = _fit_stages(st, bm, bn, bk, cg)
                            if s < 1:
                                continue
                            for c in (clusters if cg == 1 else {1}):
                                out.add((0, batched, Knobs(bm, bn, bk, s, 1, c,
                                                           cta_group=cg).as_tuple()))
                            # BatchMatMul units of several batches (bpu)
                            if batched and cg == 1 and bm == 128 and not (bk > 32 and bk % 64):
                                for u in (2, 4):
                                    if spec.b % u or 2 * u * bn > 512:
                                        continue
                                    su = _fit_stages(st, bm, bn, bk, 1, u)
                                    if su >= 1:
                                        out.add((0, batched, Knobs(bm, bn, bk, su, 1, 1, bpu=u).as_tuple()))
                            # DSMEM split-K instances compile the split in
                            # (TMA split-K for non-batched 2/4 slices) compile the split in
                            if cg == 1 and bm == 128:
                                for sp in (2, 4, 8):
                                    kn = Knobs(bm, bn, bk, s, sp, 1, batched=int(batched))
                                    if (kn.dsmem_split() or kn.tma_split()) and spec.k % (sp * bk) == 0:
                                        out.add((0, batched, kn.as_tuple()))
    elif isinstance(spec, Conv2dSpec):
        out |= _conv_instances(spec)
    return out


def prune_stale(cache_dir: str = capi.DEFAULT_CACHE) -> int:
    """Delete cubins built from an earlier kernel source (their key ends in a
    different source hash), so the cache that travels with the repo holds
    only loadable instances.  Returns how many were removed."""
    if not os.path.isdir(cache_dir):
        return 0
    live = {capi.kernel_key(0, (128, 128, 64, 4), False, False).rsplit("_", 1)[1],
            capi.kernel_key(2, (1, 16, 4, 1, 16, 4, 4, 4), False, True).rsplit("_", 1)[1]}
    n = 0
    for f in os.listdir(cache_dir):
        if f.endswith(".cubin") and f[:-len(".cubin")].rsplit("_", 1)[-1] not in live:
            os.remove(os.path.join(cache_dir, f))
            n += 1
    return n


def prebuild_ops(ops, cache_dir: str = capi.DEFAULT_CACHE, threads: int | None = None,
                 verbose: bool = True) -> dict:
    todo = set()
    for op in ops:
        # "tf32x3:<operator>" selects the fp32 3xTF32 family of that operator
        dtype, name = ("tf32x3", op[len("tf32x3:"):]) if op.startswith("tf32x3:") else ("bf16", op)
        todo |= family_instances(parse_operator(name), dtype)
    # dedupe by compile key (split is a launch argument)
    keyed = {}
    for fam, batched, kn in todo:
        keyed[capi.kernel_key(fam, kn, batched, fam == FAMILY_TF32X3)] = (fam, batched, kn)
    os.makedirs(cache_dir, exist_ok=True)
    pruned = prune_stale(cache_dir)
    have = set(os.listdir(cache_dir))
    pending = [v for k, v in keyed.items() if k + ".cubin" not in have]
    t0 = time.perf_counter()
    failures = []

    def one(item):
        fam, batched, kn = item
        try:
            return capi.compile_kernel(fam, kn, batched, fam == FAMILY_TF32X3, cache_dir)
        except capi.OpevoError as err:
            failures.append((item, str(err)[:200]))
            return 0.0

    nthreads = threads or min(16, os.cpu_count() or 1)
    with ThreadPoolExecutor(nthreads) as pool:
        ms = list(pool.map(one, pending))
    stats = {"instances": len(keyed), "compiled": len(pending) - len(failures), "pruned": pruned,
             "failed": len(failures), "compile_s_total": sum(ms) / 1e3,
             "wall_s": time.perf_counter() - t0}
    if verbose:
        print(f"[prebuild] {stats}")
        for f in failures[:5]:
            print("[prebuild] failure:", f)
    return stats
