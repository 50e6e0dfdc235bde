"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or
as the timed CPU baseline.  The product (``paper_2006_05664_b200``) never
imports it.

Contents:
* ``opevo_oracle.c`` -> ``_build/liboracle.so``: bit-exact synthetic operands
  and fp64 MatMul / BMM / Conv2d (paper definitions);
* ``opevo_port.py``: a compact restatement of the reference's OpEvo loop and
  synthetic CPU evaluator (reference pkg/src/topotune/engine.py,
  benchmarks.py), pinned by tests/golden (trajectory hashes frozen from the
  reference) -- the CPU arm of bench.py.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "opevo_oracle.c")
LIB = os.path.join(HERE, "_build", "liboracle.so")

_lib = None


def build() -> str:
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", LIB, SRC, "-lm"])
    return LIB


def load():
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(LIB)
        fp, dp = C.POINTER(C.c_float), C.POINTER(C.c_double)
        lib.oracle_fill.argtypes = [fp, C.c_uint64, C.c_uint64, C.c_int]
        lib.oracle_fill_bf16_bits.argtypes = [C.POINTER(C.c_uint16), C.c_uint64, C.c_uint64]
        lib.oracle_gemm.argtypes = [fp, fp, dp, C.c_int64, C.c_int64, C.c_int64, C.c_int64]
        lib.oracle_gemm_rows.argtypes = [fp, fp, dp, C.c_int64, C.c_int64, C.c_int64,
                                         C.POINTER(C.c_int64), C.c_int64]
        lib.oracle_conv.argtypes = [fp, fp, dp] + [C.c_int] * 9
        lib.oracle_compare.argtypes = [fp, dp, C.c_uint64, dp, dp, C.POINTER(C.c_uint64)]
        for f in (lib.oracle_fill, lib.oracle_fill_bf16_bits, lib.oracle_gemm, lib.oracle_gemm_rows,
                  lib.oracle_conv, lib.oracle_compare):
            f.restype = None
        _lib = lib
    return _lib


def _fp(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def operand(n: int, seed: int, bf16: bool = True):
    """The evaluator's synthetic operand (values as float32)."""
    import numpy as np

    out = np.empty(n, dtype=np.float32)
    load().oracle_fill(_fp(out), n, seed, int(bf16))
    return out


def operand_bf16_bits(n: int, seed: int):
    import numpy as np

    out = np.empty(n, dtype=np.uint16)
    load().oracle_fill_bf16_bits(out.ctypes.data_as(C.POINTER(C.c_uint16)), n, seed)
    return out


def gemm(a, b, batch: int, rows: int, cols: int, depth: int):
    """fp64 R[b][r][c] = sum_k A[b][r][k] B[b][c][k] (B K-major)."""
    import numpy as np

    out = np.empty(batch * rows * cols, dtype=np.float64)
    load().oracle_gemm(_fp(a), _fp(b), _dp(out), batch, rows, cols, depth)
    return out


def gemm_rows(a, b, rows: int, cols: int, depth: int, row_idx):
    """fp64 rows ``row_idx`` (counted over all batches, b * rows + r) of
    :func:`gemm`: an array [len(row_idx)][cols]."""
    import numpy as np

    idx = np.ascontiguousarray(row_idx, dtype=np.int64)
    out = np.empty(len(idx) * cols, dtype=np.float64)
    load().oracle_gemm_rows(_fp(a), _fp(b), _dp(out), rows, cols, depth,
                            idx.ctypes.data_as(C.POINTER(C.c_int64)), len(idx))
    return out.reshape(len(idx), cols)


def conv(x, w, n, c, h, wd, k, kh, kw, stride, pad):
    """fp64 direct conv of NCHW x OIHW -> NHWC."""
    import numpy as np

    ho = (h + 2 * pad - kh) // stride + 1
    wo = (wd + 2 * pad - kw) // stride + 1
    out = np.empty(n * ho * wo * k, dtype=np.float64)
    load().oracle_conv(_fp(x), _fp(w), _dp(out), n, c, h, wd, k, kh, kw, stride, pad)
    return out


def compare(c_vals, ref):
    """(max|C-R|, max|R|, non-finite count)."""
    import numpy as np

    md, mr, bad = C.c_double(), C.c_double(), C.c_uint64()
    c_vals = np.ascontiguousarray(c_vals, dtype=np.float32)
    ref = np.ascontiguousarray(ref, dtype=np.float64)
    load().oracle_compare(_fp(c_vals), _dp(ref), len(ref), C.byref(md), C.byref(mr), C.byref(bad))
    return md.value, mr.value, bad.value
