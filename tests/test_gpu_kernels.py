"""GPU parity of the sm_100a kernel family, through the C ABI.

Each kernel instance is checked three ways on the same synthetic inputs:
1. in-library against the independent SIMT fp32 reference (the evaluator's
   own verification, tolerance 1e-2 relative for bf16 outputs);
2. the downloaded output against the CPU fp64 oracle (oracle/, bit-identical
   operands regenerated on the host) -- bf16 tolerance 1e-2 relative to
   max|R| (north star: "bf16 within 1e-2 relative");
3. the in-library reference itself against the oracle (fp32 accumulation vs
   fp64: 1e-5 relative).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

BF16_TOL = 1e-2
REF_TOL = 1e-5


@pytest.fixture(scope="module")
def dev():
    from paper_2006_05664_b200 import capi

    d = capi.Device(0)
    yield d
    d.close()


def _oracle_gemm(batch, rows, cols, depth, seed):
    import oracle

    a = oracle.operand(batch * rows * depth, seed)
    b = oracle.operand(batch * cols * depth, seed + 1)
    return oracle.gemm(a, b, batch, rows, cols, depth)


def _rel(out, ref):
    import oracle

    md, mr, bad = oracle.compare(out, ref)
    assert bad == 0, f"{bad} non-finite outputs"
    return md / mr


def test_device_is_b200(dev):
    assert dev.cc == (10, 0)
    assert dev.sm_count == 148


GEMM_CASES = [
    # (rows, cols, depth, knobs = bm, bn, bk, stages, split, cluster)
    (256, 256, 256, (128, 128, 64, 4, 1, 1)),
    (512, 1024, 1024, (128, 128, 64, 4, 1, 1)),
    (512, 1024, 1024, (128, 64, 128, 3, 1, 1)),
    (512, 1024, 1024, (256, 128, 64, 4, 1, 1)),
    (512, 1024, 1024, (128, 256, 64, 3, 1, 1)),
    (512, 1024, 1024, (128, 32, 32, 6, 1, 1)),
    (512, 960, 1024, (128, 48, 16, 8, 1, 1)),
    (512, 960, 1024, (128, 48, 64, 4, 1, 1)),
    (512, 960, 1024, (128, 80, 64, 4, 1, 1)),
    (512, 1024, 1024, (128, 64, 16, 8, 1, 1)),
    (512, 1024, 1024, (128, 64, 32, 6, 1, 1)),
    (512, 1024, 1024, (128, 16, 64, 4, 1, 1)),
    (512, 1024, 1024, (128, 64, 256, 2, 1, 1)),
    (512, 1024, 1024, (128, 128, 64, 4, 2, 1)),
    (512, 1024, 1024, (128, 128, 64, 4, 4, 1)),
    (512, 1024, 1024, (128, 64, 64, 4, 1, 2)),
    (512, 1024, 1024, (128, 64, 64, 4, 1, 4)),
    (512, 1024, 1024, (256, 64, 64, 4, 2, 2)),
    (1024, 1024, 1024, (128, 128, 64, 4, 1, 1)),
    # CTA pairs (cta_group::2): knobs ..., tile_h, tile_w, acc, cta_group
    (512, 1024, 1024, (256, 128, 64, 4, 1, 1, 1, 1, 1, 2)),
    (512, 1024, 1024, (256, 64, 128, 4, 1, 1, 1, 1, 1, 2)),
    (512, 1024, 1024, (256, 256, 64, 4, 1, 1, 1, 1, 1, 2)),
    (512, 1024, 1024, (256, 32, 64, 6, 2, 1, 1, 1, 1, 2)),
    (1024, 1024, 1024, (256, 128, 128, 3, 2, 1, 1, 1, 2, 2)),
    # persistent grid with a K-split last wave (stream-K style tail), and the
    # one-CTA-per-tile grid (knob 10 = 1)
    (2048, 2048, 512, (128, 64, 64, 4, 1, 1, 1, 1, 1, 1, 2)),
    (2048, 4096, 256, (256, 128, 64, 4, 1, 1, 1, 1, 1, 2, 2)),
    (2048, 4096, 256, (256, 128, 64, 4, 1, 1, 1, 1, 1, 2)),
    (2048, 2048, 512, (128, 64, 64, 4, 1, 1, 1, 1, 1, 1, 1)),
    (2048, 2048, 512, (256, 256, 64, 3, 1, 1, 1, 1, 1, 1, 0)),
    # TMA split-K (2 or 4 slices, one wave: fp32 partials through TMA)
    (512, 1024, 1024, (128, 128, 64, 4, 2)),
    (512, 1024, 1024, (128, 128, 64, 4, 4)),
    (1024, 1024, 1024, (128, 128, 128, 3, 2)),
    (512, 1024, 1024, (128, 256, 64, 3, 2)),
    # DSMEM split-K (the K slices of a tile form a cluster, reduce in smem)
    (512, 1024, 1024, (128, 32, 64, 4, 8)),
    (512, 960, 1024, (128, 48, 64, 4, 2)),
    # split 16 falls back to the global-memory reduction
    (512, 1024, 1024, (128, 64, 64, 2, 16)),
    # K-interleaved accumulators
    (512, 1024, 1024, (128, 64, 128, 3, 1, 1, 1, 1, 4, 1)),
    (512, 1024, 1024, (256, 64, 64, 3, 1, 1, 1, 1, 2, 1)),
]


@pytest.mark.parametrize("rows,cols,depth,knobs", GEMM_CASES)
def test_matmul_parity(dev, rows, cols, depth, knobs):
    from paper_2006_05664_b200 import capi

    op = dev.prepare(capi.MATMUL, rows=rows, cols=cols, depth=depth, seed=1234)
    try:
        t = dev.trial(op, knobs, warmup=1, reps=3, tol=BF16_TOL)
        assert t.ok, t.message
        assert t.rel_err < BF16_TOL
        assert t.tflops > 0
        ref = _oracle_gemm(1, rows, cols, depth, 1234)
        assert _rel(op.output(), ref) < BF16_TOL
        assert _rel(op.reference(), ref) < REF_TOL
    finally:
        op.close()


@pytest.mark.parametrize("knobs", [(128, 64, 64, 2, 1, 1), (128, 64, 64, 2, 2, 1), (128, 64, 32, 4, 4, 1),
                                   (128, 32, 64, 4, 1, 2), (256, 64, 64, 3, 1, 1, 1, 1, 1, 2),
                                   # several batches per work unit (knob 12)
                                   (128, 64, 128, 2, 1, 1, 1, 1, 1, 1, 0, 0, 2),
                                   (128, 64, 64, 2, 1, 1, 1, 1, 1, 1, 0, 0, 4),
                                   (128, 32, 32, 4, 1, 1, 1, 1, 1, 1, 0, 0, 4)])
def test_batchmatmul_parity(dev, knobs):
    from paper_2006_05664_b200 import capi

    b, n, m, k = 12, 256, 64, 128     # BMM1-like per-batch shape
    op = dev.prepare(capi.BATCHMATMUL, batch=b, rows=n, cols=m, depth=k, seed=77)
    try:
        t = dev.trial(op, knobs, warmup=1, reps=3)
        assert t.ok, t.message
        ref = _oracle_gemm(b, n, m, k, 77)
        assert _rel(op.output(), ref) < BF16_TOL
    finally:
        op.close()


@pytest.mark.parametrize("knobs", [
    (128, 64, 64, 4, 1, 1, 8, 8),
    (128, 32, 64, 3, 1, 1, 4, 8),
    (128, 64, 32, 6, 3, 1, 2, 8),
    (128, 64, 64, 4, 1, 1, 1, 8),
    # weight-resident panel (knob 11): stages carry activations only
    (128, 64, 64, 4, 1, 1, 8, 8, 1, 1, 0, 1),
    (128, 64, 64, 3, 1, 1, 4, 2, 1, 1, 0, 1),
    (128, 64, 64, 6, 1, 1, 8, 8, 1, 1, 0, 1),
    # 256-pixel tiles (two M=128 atoms per K step), streaming and resident
    (256, 64, 64, 4, 1, 1, 8, 8),
    (256, 64, 64, 3, 1, 1, 8, 8, 1, 1, 0, 1),
    (256, 32, 64, 4, 3, 1, 4, 8),
])
def test_conv2d_parity(dev, knobs):
    import oracle
    from paper_2006_05664_b200 import capi

    n, c, h, w, k, kh, kw, s, p = 16, 64, 16, 16, 64, 3, 3, 1, 1
    op = dev.prepare(capi.CONV2D, conv=[n, c, h, w, k, kh, kw, s, p], seed=5)
    try:
        t = dev.trial(op, knobs, warmup=1, reps=3)
        assert t.ok, t.message
        x = oracle.operand(n * c * h * w, 5)
        f = oracle.operand(k * c * kh * kw, 6)
        ref = oracle.conv(x, f, n, c, h, w, k, kh, kw, s, p)
        assert _rel(op.output(), ref) < BF16_TOL
        assert _rel(op.reference(), ref) < REF_TOL
    finally:
        op.close()


@pytest.mark.parametrize("knobs", [
    # halo lines (TILE_W = 17 - KW = 14 pixels per 16-row line, one TMA box
    # per filter row serving its three taps): streaming and resident weights,
    # 128- and 256-row tiles, 2-row line blocks, BN 32
    (128, 64, 64, 4, 1, 1, 4, 14),
    (128, 64, 64, 4, 1, 1, 4, 14, 1, 1, 0, 1),
    (256, 64, 64, 3, 1, 1, 4, 14),
    (256, 64, 64, 3, 1, 1, 2, 14, 1, 1, 0, 1),
    (128, 64, 64, 4, 1, 1, 2, 14),
    (128, 32, 64, 4, 1, 1, 4, 14),
])
def test_conv2d_halo_lines_parity(dev, knobs):
    import oracle
    from paper_2006_05664_b200 import capi

    n, c, h, w, k, kh, kw, s, p = 8, 64, 28, 28, 64, 3, 3, 1, 1
    op = dev.prepare(capi.CONV2D, conv=[n, c, h, w, k, kh, kw, s, p], seed=5)
    try:
        t = dev.trial(op, knobs, warmup=1, reps=3)
        assert t.ok, t.message
        x = oracle.operand(n * c * h * w, 5)
        f = oracle.operand(k * c * kh * kw, 6)
        ref = oracle.conv(x, f, n, c, h, w, k, kh, kw, s, p)
        assert _rel(op.output(), ref) < BF16_TOL
    finally:
        op.close()


def test_conv2d_halo_lines_wide_cin(dev):
    """Cin = 128 > BK: two channel blocks per filter row, weight tiles loaded
    one 2-D box per tap (the one-box-per-row load needs Cin = BK = 64)."""
    import oracle
    from paper_2006_05664_b200 import capi

    n, c, h, w, k, kh, kw, s, p = 4, 128, 28, 28, 64, 3, 3, 1, 1
    op = dev.prepare(capi.CONV2D, conv=[n, c, h, w, k, kh, kw, s, p], seed=5)
    try:
        for knobs in [(128, 64, 64, 4, 1, 1, 4, 14), (128, 64, 64, 2, 1, 1, 4, 14, 1, 1, 0, 1)]:
            t = dev.trial(op, knobs, warmup=1, reps=3)
            assert t.ok, t.message
            x = oracle.operand(n * c * h * w, 5)
            f = oracle.operand(k * c * kh * kw, 6)
            ref = oracle.conv(x, f, n, c, h, w, k, kh, kw, s, p)
            assert _rel(op.output(), ref) < BF16_TOL
    finally:
        op.close()


def test_conv2d_halo_lines_need_matching_filter(dev):
    """A 14-pixel halo line is a 3-wide filter's; other filters reject it."""
    from paper_2006_05664_b200 import capi

    op = dev.prepare(capi.CONV2D, conv=[8, 64, 28, 28, 64, 5, 5, 1, 2], seed=5)
    try:
        t = dev.trial(op, (128, 64, 64, 4, 1, 1, 4, 14), warmup=1, reps=3)
        assert t.status == capi.INVALID_CONFIG, t.message
    finally:
        op.close()


F32_TOL = 1e-4   # north star: fp32 within 1e-4 relative


@pytest.mark.parametrize("knobs", [
    # SIMT family: (n2, n3, n4, m2, m3, m4, k2, k3) -- the paper's dense schedule
    (1, 16, 4, 1, 16, 4, 4, 4),
    (2, 8, 4, 2, 16, 2, 8, 2),
    (1, 32, 1, 1, 32, 1, 16, 1),
    (4, 8, 2, 1, 8, 8, 2, 8),
    (1, 4, 8, 2, 32, 4, 1, 16),
])
def test_fp32_simt_matmul_parity(dev, knobs):
    """cfg1 shape MM1 (512 x 1024 x 1024, fp32)."""
    import oracle
    from paper_2006_05664_b200 import capi

    rows, cols, depth = 512, 1024, 1024
    op = dev.prepare(capi.MATMUL, dtype=capi.F32, rows=rows, cols=cols, depth=depth, seed=31)
    try:
        t = dev.trial(op, knobs, warmup=1, reps=3, tol=F32_TOL)
        assert t.ok, t.message
        a = oracle.operand(rows * depth, 31, bf16=False)
        b = oracle.operand(cols * depth, 32, bf16=False)
        ref = oracle.gemm(a, b, 1, rows, cols, depth)
        assert _rel(op.output(), ref) < F32_TOL
    finally:
        op.close()


def test_fp32_simt_batched(dev):
    import oracle
    from paper_2006_05664_b200 import capi

    b_, n, m, k = 6, 128, 64, 128
    op = dev.prepare(capi.BATCHMATMUL, dtype=capi.F32, batch=b_, rows=n, cols=m, depth=k, seed=41)
    try:
        t = dev.trial(op, (1, 16, 4, 1, 16, 4, 4, 4), warmup=1, reps=3, tol=F32_TOL)
        assert t.ok, t.message
        ref = oracle.gemm(oracle.operand(b_ * n * k, 41, bf16=False),
                          oracle.operand(b_ * m * k, 42, bf16=False), b_, n, m, k)
        assert _rel(op.output(), ref) < F32_TOL
    finally:
        op.close()


X3_CASES = [
    # fp32 on the tensor cores (3xTF32); knobs as the tcgen05 family, BK in
    # fp32 elements: (rows, cols, depth, (bm, bn, bk, stages, split, ...))
    (512, 1024, 1024, (128, 64, 32, 4)),
    (512, 1024, 1024, (128, 128, 32, 3)),
    (512, 1024, 1024, (256, 64, 32, 2)),          # two M=128 atoms per K step
    (512, 1024, 1024, (128, 64, 16, 6)),          # 64-byte swizzle
    (512, 1024, 1024, (128, 64, 8, 8)),           # 32-byte swizzle
    (512, 1024, 1024, (128, 32, 64, 2)),          # two swizzle atoms per stage
    (512, 1024, 1024, (128, 64, 32, 4, 2)),       # DSMEM split-K
    (512, 1024, 1024, (128, 64, 32, 3, 4)),
    (512, 1024, 1024, (128, 64, 32, 3, 16)),      # global split-K reduction
    (2048, 2048, 512, (128, 64, 32, 4, 1, 1, 1, 1, 1, 1, 0)),   # persistent: 512 tiles
    (1024, 1024, 1024, (128, 128, 32, 3, 1, 1, 1, 1, 1, 1, 1)),
]


@pytest.mark.parametrize("rows,cols,depth,knobs", X3_CASES)
def test_fp32_tf32x3_matmul_parity(dev, rows, cols, depth, knobs):
    """fp32 MatMul on tcgen05 (kind::tf32 x3) within the fp32 tolerance of
    the north star, against the fp64 oracle on the same fp32 operands."""
    import oracle
    from paper_2006_05664_b200 import capi

    op = dev.prepare(capi.MATMUL, dtype=capi.F32_TF32X3, rows=rows, cols=cols, depth=depth, seed=31)
    try:
        t = dev.trial(op, knobs, warmup=1, reps=3, tol=F32_TOL)
        assert t.ok, t.message
        assert t.rel_err < F32_TOL
        a = oracle.operand(rows * depth, 31, bf16=False)
        b = oracle.operand(cols * depth, 32, bf16=False)
        ref = oracle.gemm(a, b, 1, rows, cols, depth)
        assert _rel(op.output(), ref) < F32_TOL
    finally:
        op.close()


def test_fp32_tf32x3_batched(dev):
    import oracle
    from paper_2006_05664_b200 import capi

    b_, n, m, k = 12, 256, 64, 128
    op = dev.prepare(capi.BATCHMATMUL, dtype=capi.F32_TF32X3, batch=b_, rows=n, cols=m, depth=k, seed=41)
    try:
        for knobs in [(128, 64, 32, 4), (128, 32, 16, 4, 2)]:
            t = dev.trial(op, knobs, warmup=1, reps=3, tol=F32_TOL)
            assert t.ok, t.message
            ref = oracle.gemm(oracle.operand(b_ * n * k, 41, bf16=False),
                              oracle.operand(b_ * m * k, 42, bf16=False), b_, n, m, k)
            assert _rel(op.output(), ref) < F32_TOL
    finally:
        op.close()


def test_fp32_tf32x3_rejects_bf16_only_knobs(dev):
    """CTA pairs, multicast clusters and batches per unit are bf16-only."""
    from paper_2006_05664_b200 import capi

    op = dev.prepare(capi.MATMUL, dtype=capi.F32_TF32X3, rows=512, cols=1024, depth=1024, seed=31)
    try:
        for knobs in [(256, 64, 32, 2, 1, 1, 1, 1, 1, 2), (128, 64, 32, 2, 1, 2)]:
            t = dev.trial(op, knobs, warmup=1, reps=3, tol=F32_TOL)
            assert t.status == capi.INVALID_CONFIG, (knobs, t.message)
    finally:
        op.close()


def test_invalid_knobs_score_invalid(dev):
    from paper_2006_05664_b200 import capi

    op = dev.prepare(capi.MATMUL, rows=512, cols=512, depth=512)
    try:
        for knobs in [(96, 128, 64, 4, 1, 1), (128, 128, 64, 40, 1, 1), (128, 512, 64, 2, 1, 1),
                      (128, 192, 64, 4, 1, 1)]:
            t = dev.trial(op, knobs)
            assert t.status == capi.INVALID_CONFIG, (knobs, t)
    finally:
        op.close()


def test_cold_and_warm_timing(dev):
    from paper_2006_05664_b200 import capi

    op = dev.prepare(capi.MATMUL, rows=1024, cols=1024, depth=1024)
    try:
        k = dev.kernel(op, (128, 128, 64, 4, 1, 1))
        warm = k.time(warmup=3, reps=20, flush_l2=False)
        cold = k.time(warmup=1, reps=5, flush_l2=True)
        assert 0 < warm < 1.0 and 0 < cold < 1.0
        k.close()
    finally:
        op.close()


def test_timing_modes_agree(dev):
    """Graph (0), cold-L2 (1) and gated-stream (2) timings of one instance are
    all positive; the gated stream launches sit within 2x of the graph."""
    from paper_2006_05664_b200 import capi

    op = dev.prepare(capi.MATMUL, rows=1024, cols=1024, depth=1024)
    try:
        k = dev.kernel(op, (128, 64, 128, 3, 1, 1))
        g = k.time(warmup=3, reps=20, flush_l2=0)
        s = k.time(warmup=3, reps=20, flush_l2=2)
        c = k.time(warmup=1, reps=3, flush_l2=1)
        assert 0 < g < 1.0 and 0 < s < 1.0 and 0 < c < 1.0
        assert 0.5 < s / g < 2.0
        k.close()
    finally:
        op.close()


def test_trial_batch_matches_single_trials(dev):
    """opevo_trial_batch: per-trial statuses equal opevo_trial's (valid,
    invalid, split-K and CTA-pair instances mixed), every verified output
    within tolerance, and the last instance's output matches the oracle."""
    from paper_2006_05664_b200 import capi

    rows, cols, depth = 512, 1024, 1024
    knob_list = [(128, 64, 128, 3, 1, 1), (96, 128, 64, 4, 1, 1), (128, 128, 64, 4, 2, 1),
                 (256, 64, 128, 4, 1, 1, 1, 1, 1, 2), (128, 512, 64, 2, 1, 1), (128, 32, 64, 4, 1, 2)]
    op = dev.prepare(capi.MATMUL, rows=rows, cols=cols, depth=depth, seed=1234)
    try:
        batch = dev.trial_batch(op, knob_list, warmup=2, reps=5)
        single = [dev.trial(op, kn, warmup=2, reps=5) for kn in knob_list]
        assert [t.status for t in batch] == [t.status for t in single]
        for t in batch:
            if t.ok:
                assert t.rel_err < BF16_TOL and t.tflops > 0 and t.ms > 0
            else:
                assert t.status == capi.INVALID_CONFIG and t.message
        last = dev.trial_batch(op, [knob_list[3]], warmup=1, reps=3)[0]
        assert last.ok
        assert _rel(op.output(), _oracle_gemm(1, rows, cols, depth, 1234)) < BF16_TOL
    finally:
        op.close()


def test_trial_batch_verification_cache(dev):
    """A trial of an instance already verified on the same operands is
    re-timed without re-running the check (verify_cached = 1, the earlier
    rel_err, one fewer compare kernel); new operands clear the cache."""
    import ctypes

    from paper_2006_05664_b200 import capi

    rows, cols, depth = 512, 1024, 1024
    kn = [(128, 64, 128, 3, 1, 1), (128, 128, 64, 4, 2, 1)]
    op = dev.prepare(capi.MATMUL, rows=rows, cols=cols, depth=depth, seed=1234)
    try:
        first = dev.trial_batch(op, kn, warmup=3, reps=5, flush_l2=2)
        again = dev.trial_batch(op, kn, warmup=3, reps=5, flush_l2=2)
        assert all(t.ok and not t.verify_cached for t in first)
        assert all(t.ok and t.verify_cached for t in again)
        assert [t.rel_err for t in again] == [t.rel_err for t in first]
        # the re-timed launches still produce the verified output
        assert _rel(op.output(), _oracle_gemm(1, rows, cols, depth, 1234)) < BF16_TOL
        # the same number of tuned-kernel launches (the check launch becomes a warm-up)
        assert [t.launches for t in again] == [t.launches for t in first]
        a = (ctypes.c_char * op.a_bytes)()
        b = (ctypes.c_char * op.b_bytes)()
        op.read_inputs(ctypes.addressof(a), ctypes.addressof(b))
        op.upload(ctypes.addressof(a), ctypes.addressof(b))
        fresh = dev.trial_batch(op, kn, warmup=3, reps=5, flush_l2=2)
        assert all(t.ok and not t.verify_cached for t in fresh)
    finally:
        op.close()


@pytest.mark.parametrize("op_id", ["matmul:1024,1024,1024", "batchmatmul:960,128,64,128",
                                   "conv2d:32,64,56,56,64,3,3,1,1"])
def test_mapping_smem_matches_library(dev, op_id):
    """The mapping's shared-memory accounting (stage fitting) equals what the
    library requests at launch for every sampled valid configuration."""
    from paper_2006_05664_b200.evaluator import _op_args
    from paper_2006_05664_b200.mapping import config_to_knobs, gpu_operator_space
    from paper_2006_05664_b200.operators import parse_operator

    spec = parse_operator(op_id)
    space = gpu_operator_space(spec)
    op = dev.prepare(**_op_args(spec))
    rng = np.random.default_rng(3)
    seen = 0
    try:
        for _ in range(3000):
            m = config_to_knobs(spec, space, space.sample_uniform(rng))
            if not m.valid:
                continue
            k = dev.kernel(op, m.knobs.as_tuple())
            assert k.info.smem_bytes == m.knobs.smem_bytes(), (m.knobs, k.info.smem_bytes)
            k.close()
            seen += 1
            if seen >= 40:
                break
        assert seen >= 10
    finally:
        op.close()


def test_slow_candidate_is_timed_by_its_verified_launch(dev):
    """A candidate whose verified launch alone exceeds the per-trial device
    budget (0.3 ms) gets no further launches: one launch, positive time."""
    from paper_2006_05664_b200 import capi

    op = dev.prepare(capi.MATMUL, rows=4096, cols=4096, depth=4096)
    try:
        t = dev.trial(op, (128, 16, 32, 2, 1, 1))
        assert t.ok, t.message
        assert t.launches == 1 and t.ms > 0.3
        fast = dev.trial(op, (256, 256, 64, 4, 1, 1, 1, 1, 1, 2))
        assert fast.ok and fast.launches > 3 and fast.ms < 0.3
        b = dev.trial_batch(op, [(128, 16, 32, 2, 1, 1), (256, 256, 64, 4, 1, 1, 1, 1, 1, 2)])
        assert [x.launches == 1 for x in b] == [True, False]
    finally:
        op.close()


def test_trial_batch_gated_stream_mode(dev):
    """Mode 2 (the default fitness timing): every verified instance timed
    behind shared device gates with one synchronisation; statuses as in
    mode 0 and times within 2x of the graph timing."""
    from paper_2006_05664_b200 import capi

    op = dev.prepare(capi.MATMUL, rows=1024, cols=1024, depth=1024, seed=1234)
    try:
        kl = [(128, 64, 128, 3, 1, 1), (128, 128, 64, 4, 1, 1), (96, 128, 64, 4, 1, 1),
              (256, 64, 128, 4, 1, 1, 1, 1, 1, 2)] * 4          # > 64 launches: several gates
        s = dev.trial_batch(op, kl, warmup=3, reps=20, flush_l2=2)
        g = dev.trial_batch(op, kl, warmup=3, reps=20, flush_l2=0)
        assert [t.status for t in s] == [t.status for t in g]
        for a, b in zip(s, g):
            if a.ok:
                assert 0.5 < a.ms / b.ms < 2.0 and a.rel_err < BF16_TOL
    finally:
        op.close()
