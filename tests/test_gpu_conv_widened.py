"""Conv2d beyond stride-1 power-of-two tiles, against the fp64 oracle.

* The paper's own AlexNet convolutions: C1 (512, 3, 227,
  227) * (64, 3, 11, 11), stride 4, pad 0 -- Cin = 3 padded to 16 in the
  kernel layout, the activation tensor map traversing W and H with element
  stride 4 -- and C2 (512, 64, 27, 27) * (192, 64, 5, 5), pad 2, whose 27-pixel
  rows tile as padded lines.  Exact shapes, four whole images checked.
* Strided dense tiles, split over filter taps with padded lines, and CTA
  pairs (cta_group::2) on the BASELINE conv (cfg4, full output).

Every instance here comes from the mapping (mapping.config_to_knobs), so
what is tested is what the search can reach.  Tolerance: bf16 1e-2 of max|R|.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

BF16_TOL = 1e-2
SEED = 4321


@pytest.fixture(scope="module")
def dev():
    from paper_2006_05664_b200 import capi

    d = capi.Device(0)
    yield d
    d.close()


def _rel(out, ref):
    import oracle

    md, mr, bad = oracle.compare(out, ref)
    assert bad == 0, f"{bad} non-finite outputs"
    return md / mr


def _knobs(op_id, cfg):
    from paper_2006_05664_b200.mapping import config_to_knobs, gpu_operator_space
    from paper_2006_05664_b200.operators import parse_operator

    spec = parse_operator(op_id)
    m = config_to_knobs(spec, gpu_operator_space(spec), cfg)
    assert m.valid, m.reason
    return m.knobs.as_tuple()


def _check_images(dev, op_id, cfgs, images):
    """Run each mapped instance on the exact operator; compare whole images
    (NHWC output rows of those images) with the fp64 oracle."""
    import oracle
    from paper_2006_05664_b200 import capi
    from paper_2006_05664_b200.operators import parse_operator

    spec = parse_operator(op_id)
    n, c, h, w = spec.batch, spec.in_channels, spec.in_height, spec.in_width
    k, kh, kw, s, p = spec.out_channels, spec.kernel_h, spec.kernel_w, spec.stride, spec.padding
    ho, wo = spec.out_height, spec.out_width
    x = oracle.operand(n * c * h * w, SEED).reshape(n, c * h * w)
    f = oracle.operand(k * c * kh * kw, SEED + 1)
    refs = {i: oracle.conv(np.ascontiguousarray(x[i]), f, 1, c, h, w, k, kh, kw, s, p) for i in images}
    op = dev.prepare(capi.CONV2D, conv=[n, c, h, w, k, kh, kw, s, p], seed=SEED)
    try:
        for cfg in cfgs:
            knobs = _knobs(op_id, cfg)
            t = dev.trial(op, knobs, warmup=1, reps=2)
            assert t.ok, (knobs, t.message)
            # FLOPs use the operator's Cin, not the padded one
            assert abs(t.tflops * t.ms * 1e9 / spec.flops() - 1.0) < 1e-6
            out = op.output().reshape(n, ho * wo * k)
            for i in images:
                assert _rel(out[i], refs[i]) < BF16_TOL, (knobs, i)
    finally:
        op.close()


C1 = "conv2d:512,3,227,227,64,11,11,4,0"
C2 = "conv2d:512,64,27,27,192,5,5,1,2"


def test_alexnet_c1_exact_shape(dev):
    cfgs = [
        # 11-pixel lines (of 16 rows), one line per image row, 8 images
        ((1, 1, 8, 8), (55, 1, 1, 1), (5, 1, 11, 1), (1, 3), (1, 11), (1, 11), "explicit_unroll_off", 64),
        # 5-row x 11-pixel line blocks (80 of 128 rows used), split over the 11 filter rows
        ((1, 1, 8, 8), (11, 1, 5, 1), (5, 1, 11, 1), (1, 3), (11, 1), (1, 11), "explicit_unroll_off", 512),
        # 256-pixel tiles (two M = 128 atoms), 5-pixel lines, BN 32
        ((2, 2, 4, 4), (55, 1, 1, 1), (11, 1, 5, 1), (1, 3), (1, 11), (1, 11), "explicit_unroll_off", 1500),
    ]
    _check_images(dev, C1, cfgs, images=(0, 137, 400, 511))


def test_alexnet_c2_exact_shape(dev):
    cfgs = [
        # 27-pixel lines of 32 rows, 256-pixel tiles, BN 64
        ((3, 2, 4, 8), (27, 1, 1, 1), (1, 3, 3, 3), (1, 64), (1, 5), (1, 5), "explicit_unroll_off", 512),
        # 9-pixel lines of 16 rows, BN 192 (UMMA N = 192), BK 32
        ((1, 1, 8, 24), (27, 1, 1, 1), (3, 1, 3, 3), (2, 32), (1, 5), (1, 5), "explicit_unroll_off", 64),
        # 3 lines x 9 pixels, split over the 5 filter rows (global reduction skips junk rows)
        ((3, 1, 8, 8), (9, 1, 3, 1), (3, 1, 3, 3), (1, 64), (5, 1), (1, 5), "explicit_unroll_off", 64),
        # dense 1x1-pixel tiles of 128 images (the only dense tiling of 27 x 27)
        ((2, 1, 8, 12), (27, 1, 1, 1), (27, 1, 1, 1), (1, 64), (1, 5), (1, 5), "explicit_unroll_off", 16),
    ]
    _check_images(dev, C2, cfgs, images=(0, 255, 511))


def test_strided_dense_tiles(dev):
    """Stride 2 with dense 8x8 / 4x16 tiles and a tap split."""
    op_id = "conv2d:8,32,64,64,64,3,3,2,1"        # 32x32 outputs
    cfgs = [((1, 1, 8, 8), (4, 1, 8, 1), (4, 1, 8, 1), (1, 32), (1, 3), (1, 3), "explicit_unroll_off", 64),
            ((1, 1, 8, 8), (8, 1, 4, 1), (2, 1, 16, 1), (1, 32), (3, 1), (1, 3), "explicit_unroll_off", 16),
            ((2, 1, 4, 8), (4, 1, 8, 1), (4, 1, 8, 1), (2, 16), (1, 3), (1, 3), "explicit_unroll_on", 64)]
    _check_images(dev, op_id, cfgs, images=(0, 3, 7))


def test_conv4_cta_pairs(dev):
    """cta_group::2 on the BASELINE conv: halo lines and dense 256-pixel tiles
    on CTA pairs, full output against the oracle."""
    import oracle
    from paper_2006_05664_b200 import capi

    op_id = "conv2d:32,64,56,56,64,3,3,1,1"
    cfgs = [
        ((1, 2, 4, 8), (14, 2, 2, 1), (4, 2, 7, 1), (1, 64), (1, 3), (1, 3), "explicit_unroll_off", 64),
        ((1, 2, 4, 8), (14, 2, 2, 1), (4, 2, 7, 1), (1, 64), (1, 3), (1, 3), "explicit_unroll_off", 16),
        ((1, 2, 4, 8), (14, 2, 2, 1), (7, 1, 8, 1), (1, 64), (1, 3), (1, 3), "explicit_unroll_off", 64),
        ((2, 2, 4, 4), (7, 2, 4, 1), (7, 1, 8, 1), (1, 64), (1, 3), (1, 3), "explicit_unroll_off", 512),
    ]
    knobs = [_knobs(op_id, c) for c in cfgs]
    assert all(k[9] == 2 for k in knobs)
    n, c, h, w, k, kh, kw, s, p = 32, 64, 56, 56, 64, 3, 3, 1, 1
    ref = oracle.conv(oracle.operand(n * c * h * w, SEED), oracle.operand(k * c * kh * kw, SEED + 1),
                      n, c, h, w, k, kh, kw, s, p)
    op = dev.prepare(capi.CONV2D, conv=[n, c, h, w, k, kh, kw, s, p], seed=SEED)
    try:
        for kn in knobs:
            t = dev.trial(op, kn, warmup=1, reps=3)
            assert t.ok, (kn, t.message)
            assert _rel(op.output(), ref) < BF16_TOL, kn
    finally:
        op.close()


def test_narrow_cin_upload_round_trip(dev):
    """Cin = 3: the kernel layout is NHWC with 16 channels (13 zero); an
    upload of that layout (new operands) is converted back to the paper's
    NCHW for the reference, and the output matches the oracle."""
    import oracle
    from paper_2006_05664_b200 import capi

    n, c, h, w, k, kh, kw, s, p = 4, 3, 35, 35, 32, 5, 5, 2, 1
    op = dev.prepare(capi.CONV2D, conv=[n, c, h, w, k, kh, kw, s, p], seed=8)
    try:
        assert op.a_bytes == n * h * w * 16 * 2 and op.b_bytes == k * kh * kw * 16 * 2
        x = oracle.operand(n * c * h * w, 77)
        f = oracle.operand(k * c * kh * kw, 78)
        xh = np.zeros((n, h, w, 16), np.float32)
        xh[..., :c] = x.reshape(n, c, h, w).transpose(0, 2, 3, 1)
        fh = np.zeros((k, kh, kw, 16), np.float32)
        fh[..., :c] = f.reshape(k, c, kh, kw).transpose(0, 2, 3, 1)
        xb = (np.ascontiguousarray(xh).view(np.uint32) >> 16).astype(np.uint16)
        fb = (np.ascontiguousarray(fh).view(np.uint32) >> 16).astype(np.uint16)
        op.upload(xb.ctypes.data, fb.ctypes.data)
        ho = (h + 2 * p - kh) // s + 1                       # 17: padded lines of 32 rows
        knobs = (128, 32, 16, 4, 1, 1, 1, ho, 1, 1, 0, 0, 1, 32)
        t = dev.trial(op, knobs, warmup=1, reps=2)
        assert t.ok, t.message
        ref = oracle.conv(x, f, n, c, h, w, k, kh, kw, s, p)
        assert _rel(op.reference(), ref) < 1e-5
        assert _rel(op.output(), ref) < BF16_TOL
    finally:
        op.close()


R3 = "conv2d:32,128,28,28,128,3,3,1,1"


def test_halo_pairs_on_a_wider_conv(dev):
    """Halo-line CTA pairs away from cfg4: Cin = Cout = 128 on 28 x 28, where
    the 512-row pairs (256 rows, two M=256 atoms per CTA) run with BK = 128
    (two 64-channel atoms per K block, so the one-box weight load spans two
    atoms x three taps) and BK = 64, next to a 256-row pair with BK = 128."""
    cfgs = [((2, 4, 4, 4), (7, 2, 2, 1), (2, 2, 7, 1), (1, 128), (1, 3), (1, 3), "explicit_unroll_off", 64),
            ((2, 4, 4, 4), (7, 2, 2, 1), (2, 2, 7, 1), (2, 64), (1, 3), (1, 3), "explicit_unroll_off", 64),
            ((2, 2, 4, 8), (7, 2, 2, 1), (2, 2, 7, 1), (1, 128), (1, 3), (1, 3), "explicit_unroll_off", 64),
            ((2, 4, 4, 4), (14, 2, 1, 1), (2, 2, 7, 1), (2, 64), (1, 3), (1, 3), "explicit_unroll_off", 512)]
    assert [_knobs(R3, c)[0] for c in cfgs] == [512, 512, 256, 512]
    _check_images(dev, R3, cfgs, images=(0, 13, 31))
