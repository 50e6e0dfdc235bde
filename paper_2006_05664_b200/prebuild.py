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
        if spec.stride != 1:
            return out
        ths = [t for t in _divisors(spec.out_height) if 128 % t == 0]
        tws = [t for t in _divisors(spec.out_width) if 128 % t == 0]
        for bm, th, tw in itertools.product((128, 256), ths, tws):
            if th * tw > bm or bm % (th * tw) or spec.batch % (bm // (th * tw)):
                continue
            for bn in range(16, 257, 16):
                if spec.out_channels % bn or (bm == 256 and 2 * bn > 512):
                    continue
                for bk in _divisors(spec.in_channels):
                    if not _bk_ok(bk):
                        continue
                    for st in set(UNROLL_TO_STAGES.values()):
                        s = _fit_stages(st, bm, bn, bk)
                        if s >= 1:
                            out.add((1, False, Knobs(bm, bn, bk, s, 1, 1, th, tw).as_tuple()))
                        # weight-resident variant (unroll_explicit = on)
                        rs, panel = _conv_resident_fit(spec, bn, bk, 1, st, bm)
                        if rs:
                            out.add((1, False, Knobs(bm, bn, bk, rs, 1, 1, th, tw, b_res=1,
                                                     panel_bytes=panel).as_tuple()))
        # halo lines: 17 - KW output pixels per 16-row line (mapping._conv_halo_knobs)
        tw = 17 - spec.kernel_w
        if 1 <= tw < 16 and spec.out_width % tw == 0 and spec.padding < spec.kernel_w:
            for bm in (128, 256):
                for th in _divisors(spec.out_height):
                    if bm % (16 * th) or spec.batch % (bm // (16 * th)) or bm % (th * tw) == 0:
                        continue
                    for bn in range(16, 257, 16):
                        if spec.out_channels % bn or (bm == 256 and 2 * bn > 512):
                            continue
                        for bk in _divisors(spec.in_channels):
                            if bk % 64 or not _bk_ok(bk):
                                continue
                            for st in set(UNROLL_TO_STAGES.values()):
                                s = _fit_halo_stages(st, bm, bn, bk, spec.kernel_w)
                                if s >= 1:
                                    out.add((1, False, Knobs(bm, bn, bk, s, 1, 1, th, tw).as_tuple()))
                                rs, panel = _conv_resident_fit(spec, bn, bk, 1, st, bm)
                                if rs:
                                    out.add((1, False, Knobs(bm, bn, bk, rs, 1, 1, th, tw, b_res=1,
                                                             panel_bytes=panel).as_tuple()))
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
