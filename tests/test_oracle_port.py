"""Pin the oracle before trusting it: the CPU port of the reference tuner
reproduces the trajectories frozen from the reference (tests/golden), and the
C operator oracle agrees with numpy fp64 on the same bit-exact operands."""

import hashlib
import json
import os

import numpy as np
import pytest

import oracle
from oracle import opevo_port

HERE = os.path.dirname(os.path.abspath(__file__))
TRAJ = json.load(open(os.path.join(HERE, "golden", "trajectories.json")))


def _hash(names, log):
    body = "\n".join(json.dumps([{n: list(v) if isinstance(v, tuple) else v
                                  for n, v in zip(names, c)}, f]) for c, f in log)
    return hashlib.sha256(body.encode()).hexdigest()[:16]


@pytest.mark.parametrize("key", sorted(TRAJ["runs"]))
def test_port_matches_reference_trajectories(key):
    op, seed = key.split("|")
    names, log = opevo_port.opevo_run(op, seed=int(seed), budget=500)
    assert _hash(names, log) == TRAJ["runs"][key]["hash"]


def test_operand_generator_matches_numpy_restatement():
    # splitmix64 restated with numpy uint64 wrap-around arithmetic
    seed, n = np.uint64(1234), 1000
    i = np.arange(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = seed * np.uint64(0x9E3779B97F4A7C15) + i + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    x = (z >> np.uint64(40)).astype(np.float32) * np.float32(1.0 / 8388608.0) - np.float32(1.0)
    np.testing.assert_array_equal(oracle.operand(n, 1234, bf16=False), x)
    bits = x.view(np.uint32)
    rne = ((bits + np.uint32(0x7FFF) + ((bits >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16))
    np.testing.assert_array_equal(oracle.operand_bf16_bits(n, 1234), rne.astype(np.uint16))
    assert np.all(np.abs(x) <= 1.0)


def test_gemm_oracle_vs_numpy():
    b, r, c, k = 2, 33, 17, 40
    a = oracle.operand(b * r * k, 3)
    y = oracle.operand(b * c * k, 4)
    got = oracle.gemm(a, y, b, r, c, k).reshape(b, r, c)
    want = np.einsum("brk,bck->brc", a.reshape(b, r, k).astype(np.float64),
                     y.reshape(b, c, k).astype(np.float64))
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)


def test_conv_oracle_vs_numpy():
    n, c, h, w, k, kh, kw, s, p = 2, 3, 7, 6, 4, 3, 3, 1, 1
    x = oracle.operand(n * c * h * w, 5)
    f = oracle.operand(k * c * kh * kw, 6)
    got = oracle.conv(x, f, n, c, h, w, k, kh, kw, s, p).reshape(n, h, w, k)
    xp = np.pad(x.reshape(n, c, h, w).astype(np.float64), ((0, 0), (0, 0), (p, p), (p, p)))
    fw = f.reshape(k, c, kh, kw).astype(np.float64)
    want = np.zeros((n, h, w, k))
    for i in range(kh):
        for j in range(kw):
            want += np.einsum("nchw,kc->nhwk", xp[:, :, i:i + h, j:j + w], fw[:, :, i, j])
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)


def test_conv_oracle_strided():
    n, c, h, w, k, kh, kw, s, p = 1, 2, 9, 9, 3, 3, 3, 2, 0
    x = oracle.operand(n * c * h * w, 8)
    f = oracle.operand(k * c * kh * kw, 9)
    got = oracle.conv(x, f, n, c, h, w, k, kh, kw, s, p).reshape(n, 4, 4, k)
    xr = x.reshape(n, c, h, w).astype(np.float64)
    fr = f.reshape(k, c, kh, kw).astype(np.float64)
    for ho in range(4):
        for wo in range(4):
            patch = xr[0, :, ho * 2:ho * 2 + 3, wo * 2:wo * 2 + 3]
            np.testing.assert_allclose(got[0, ho, wo], np.einsum("chw,kchw->k", patch, fr),
                                       rtol=1e-12)
