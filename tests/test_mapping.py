"""Configuration -> kernel-knob mapping (mapping.py) and the GPU spaces."""

import numpy as np
import pytest

from paper_2006_05664_b200 import (
    BatchMatMulSpec,
    Conv2dSpec,
    EngineConfig,
    MatMulSpec,
    SearchSpace,
    matmul_space,
    parse_operator,
    run,
)
from paper_2006_05664_b200.mapping import (
    SMEM_LIMIT,
    Knobs,
    config_to_knobs,
    gpu_operator_space,
    valid_fraction,
)
from paper_2006_05664_b200.prebuild import family_instances


def test_gpu_space_extends_reference_space_in_json_format():
    spec = MatMulSpec(1024, 1024, 1024)
    sp = gpu_operator_space(spec)
    assert sp.names == ("n", "m", "k", "stages")
    assert sp.to_json()[:3] == matmul_space(spec).to_json()
    assert SearchSpace.from_json(sp.to_json()).to_json() == sp.to_json()


def test_matmul_mapping_levels(monkeypatch):
    spec = MatMulSpec(1024, 1024, 1024)
    sp = gpu_operator_space(spec)
    cfg = ((8, 2, 8, 8), (8, 4, 4, 8), (2, 8, 64), 4)
    m = config_to_knobs(spec, sp, cfg)
    assert m.valid
    # default: m[1] does not select a multicast cluster
    assert m.knobs == Knobs(bm=128, bn=128, bk=64, stages=4, split=2, cluster=1)
    monkeypatch.setenv("OPEVO_MAP_MULTICAST", "1")
    m = config_to_knobs(spec, sp, cfg)
    assert m.knobs == Knobs(bm=128, bn=128, bk=64, stages=4, split=2, cluster=4)
    # 256-row tile with an even row vthread split -> CTA pair
    pair = config_to_knobs(spec, sp, ((4, 2, 16, 8), (8, 4, 4, 8), (1, 16, 64), 4)).knobs
    assert pair.bm == 256 and pair.cta_group == 2 and pair.cluster == 1
    single = config_to_knobs(spec, sp, ((4, 1, 32, 8), (8, 4, 4, 8), (1, 16, 64), 4)).knobs
    assert single.bm == 256 and single.cta_group == 1
    # sub-tile splits do not change the kernel
    cfg2 = ((8, 128, 1, 1), (8, 1, 1, 128), (2, 8, 64), 4)
    assert config_to_knobs(spec, sp, cfg2).knobs == Knobs(128, 128, 64, 4, 2, 1)


@pytest.mark.parametrize("cfg,why", [
    (((16, 4, 4, 4), (8, 2, 8, 8), (1, 16, 64), 4), "BM=64"),
    (((8, 2, 8, 8), (2, 2, 16, 16), (1, 16, 64), 4), "BN=512"),
    (((8, 2, 8, 8), (8, 2, 8, 8), (1, 128, 8), 4), "BK=8"),
    (((8, 2, 8, 8), (8, 2, 8, 8), (2, 1, 512), 4), "BK=512"),
])
def test_infeasible_configs_are_invalid(cfg, why):
    spec = MatMulSpec(1024, 1024, 1024)
    m = config_to_knobs(spec, gpu_operator_space(spec), cfg)
    assert not m.valid and why.split("=")[0] in m.reason


def test_stages_clamped_to_shared_memory():
    spec = MatMulSpec(1024, 1024, 1024)
    sp = gpu_operator_space(spec)
    m = config_to_knobs(spec, sp, ((4, 4, 8, 8), (4, 4, 8, 8), (1, 8, 128), 8))
    assert m.valid and m.knobs.bm == 256 and m.knobs.bn == 256
    assert m.knobs.smem_bytes() <= SMEM_LIMIT
    assert m.knobs.stages < 8


def test_conv_mapping():
    spec = parse_operator("conv2d:32,64,56,56,64,3,3,1,1")
    sp = gpu_operator_space(spec)
    cfg = ((1, 2, 4, 8), (7, 1, 2, 4), (7, 2, 2, 2), (1, 64), (3, 1), (1, 3),
           "explicit_unroll_on", 64)
    m = config_to_knobs(spec, sp, cfg)
    assert m.valid and m.family == 1
    # co[1] = 2 (even): two M=128 atoms per K step -> 256-pixel tiles (8x8x4)
    assert m.knobs == Knobs(256, 64, 64, 4, 3, 1, 8, 8, family=1)
    # co[1] odd: 128-pixel tiles (8x8x2)
    m = config_to_knobs(spec, sp, ((1, 1, 8, 8),) + cfg[1:])
    assert m.valid and m.knobs == Knobs(128, 64, 64, 4, 3, 1, 8, 8, family=1)
    # explicit unroll without a tap split: the weight panel stays resident
    m = config_to_knobs(spec, sp, ((1, 1, 8, 8), (7, 1, 2, 4), (7, 2, 2, 2), (1, 64), (1, 3), (1, 3),
                                   "explicit_unroll_on", 512))
    assert m.valid and m.knobs.b_res == 1 and m.knobs.split == 1
    assert m.knobs.panel_bytes == 64 * 9 * 64 * 2 and m.knobs.smem_bytes() <= 232448


def test_conv_halo_lines_mapping():
    """wo[0] giving 14-pixel tiles (17 - KW for a 3x3 filter) selects halo
    lines: 16-row lines, TILE_N = BM / (16 * TILE_H), stages sized for the
    activation box plus the KW weight tiles of one filter row."""
    from paper_2006_05664_b200.mapping import SMEM_LIMIT

    spec = parse_operator("conv2d:32,64,56,56,64,3,3,1,1")
    sp = gpu_operator_space(spec)
    cfg = ((1, 1, 8, 8), (14, 1, 4, 1), (4, 2, 7, 1), (1, 64), (1, 3), (1, 3), "explicit_unroll_off", 64)
    m = config_to_knobs(spec, sp, cfg)
    assert m.valid, m.reason
    k = m.knobs
    assert (k.bm, k.bn, k.bk, k.tile_h, k.tile_w, k.split) == (128, 64, 64, 4, 14, 1)
    assert k.halo_kw() == 3 and k.stages == 4
    assert k.smem_bytes() == 4 * (128 + 3 * 64) * 64 * 2 + 32768 + 1280 <= SMEM_LIMIT
    # a split over taps cannot use halo lines
    bad = config_to_knobs(spec, sp, ((1, 1, 8, 8), (14, 1, 4, 1), (4, 2, 7, 1), (1, 64), (3, 1), (1, 3),
                                     "explicit_unroll_off", 64))
    assert not bad.valid
    # a 5x5 filter's halo lines are 12 pixels wide, so 14-pixel tiles are
    # padded lines for it instead (one box per tap, 16-row lines)
    spec5 = parse_operator("conv2d:32,64,56,56,64,5,5,1,2")
    sp5 = gpu_operator_space(spec5)
    cfg5 = ((1, 1, 8, 8), (14, 1, 4, 1), (4, 2, 7, 1), (1, 64), (1, 5), (1, 5), "explicit_unroll_off", 64)
    k5 = config_to_knobs(spec5, sp5, cfg5).knobs
    assert k5.line == 16 and k5.halo_kw() == 0 and (k5.tile_h, k5.tile_w) == (4, 14)


def test_conv_paper_operators_map():
    """The paper's AlexNet convolutions: C1 (Cin = 3 padded
    to 16, 11x11, stride 4) and C2 (5x5 on 27x27 outputs) map through padded
    lines and strided activation boxes; valid fractions above 1 %."""
    from paper_2006_05664_b200.mapping import conv_channels_padded, valid_fraction

    c1 = parse_operator("conv2d:512,3,227,227,64,11,11,4,0")
    sp1 = gpu_operator_space(c1)
    assert conv_channels_padded(3) == 16 and (c1.out_height, c1.out_width) == (55, 55)
    m = config_to_knobs(c1, sp1, ((1, 1, 8, 8), (55, 1, 1, 1), (5, 1, 11, 1), (1, 3), (1, 11), (1, 11),
                                  "explicit_unroll_off", 64))
    assert m.valid, m.reason
    assert (m.knobs.bk, m.knobs.tile_h, m.knobs.tile_w, m.knobs.line) == (16, 1, 11, 16)
    c2 = parse_operator("conv2d:512,64,27,27,192,5,5,1,2")
    sp2 = gpu_operator_space(c2)
    m2 = config_to_knobs(c2, sp2, ((3, 2, 4, 8), (27, 1, 1, 1), (1, 3, 3, 3), (1, 64), (1, 5), (1, 5),
                                   "explicit_unroll_off", 512))
    assert m2.valid, m2.reason
    assert (m2.knobs.bn, m2.knobs.tile_w, m2.knobs.line, m2.knobs.bm, m2.knobs.cta_group) == (64, 27, 32, 256, 1)
    assert valid_fraction(c1, sp1, 4000) > 0.01 and valid_fraction(c2, sp2, 4000) > 0.01


def test_conv_cta_pair_mapping():
    """An even co[1] (256-pixel tiles) with an even ho[1] runs on a CTA pair:
    each CTA holds 128 pixel rows and half the weight tile."""
    spec = parse_operator("conv2d:32,64,56,56,64,3,3,1,1")
    sp = gpu_operator_space(spec)
    halo = config_to_knobs(spec, sp, ((1, 2, 4, 8), (14, 2, 2, 1), (4, 2, 7, 1), (1, 64), (1, 3), (1, 3),
                                      "explicit_unroll_off", 64)).knobs
    assert (halo.bm, halo.cta_group, halo.tile_h, halo.tile_w, halo.halo_kw()) == (256, 2, 4, 14, 3)
    assert halo.smem_bytes() == halo.stages * (128 + 3 * 32) * 64 * 2 + 32768 + 1280
    dense = config_to_knobs(spec, sp, ((1, 2, 4, 8), (14, 2, 2, 1), (7, 1, 8, 1), (1, 64), (1, 3), (1, 3),
                                       "explicit_unroll_on", 64)).knobs
    assert dense.cta_group == 2 and dense.b_res == 0 and dense.bm == 256


def test_conv_512_row_pair_mapping():
    """A Cout split divisible by four (co[1] % 4 == 0) on a pair of halo tiles
    selects 512-row pairs: 256 rows (two M=256 atoms) per CTA, TILE_N twice
    the 256-row pair's; the same config off the halo path, or with
    co[1] = 2 mod 4, keeps 256 rows."""
    spec = parse_operator("conv2d:32,64,56,56,64,3,3,1,1")
    sp = gpu_operator_space(spec)
    big = config_to_knobs(spec, sp, ((1, 4, 2, 8), (14, 2, 2, 1), (4, 2, 7, 1), (1, 64), (1, 3), (1, 3),
                                     "explicit_unroll_off", 16)).knobs
    assert (big.bm, big.cta_group, big.bm_cta, big.tile_h, big.tile_w, big.halo_kw()) == (512, 2, 256, 4, 14, 3)
    assert big.smem_bytes() == big.stages * (256 + 3 * 32) * 64 * 2 + 32768 + 1280
    small = config_to_knobs(spec, sp, ((1, 2, 4, 8), (14, 2, 2, 1), (4, 2, 7, 1), (1, 64), (1, 3), (1, 3),
                                       "explicit_unroll_off", 16)).knobs
    assert (small.bm, small.cta_group) == (256, 2)
    dense = config_to_knobs(spec, sp, ((1, 4, 2, 8), (14, 2, 2, 1), (7, 1, 8, 1), (1, 64), (1, 3), (1, 3),
                                       "explicit_unroll_off", 16)).knobs
    assert (dense.bm, dense.cta_group) == (256, 2)


def test_bmm_mapping_is_batched():
    spec = BatchMatMulSpec(960, 128, 64, 128)
    sp = gpu_operator_space(spec)
    m = config_to_knobs(spec, sp, ((960, 1), (1, 2, 8, 8), (1, 1, 8, 8), (1, 2, 64), 2))
    assert m.valid and m.batched and m.knobs.bm == 128 and m.knobs.bn == 64


def test_tf32x3_mapping():
    """fp32 on the tensor cores: the tcgen05 mapping with BK = k[2] fp32
    elements, single-CTA tiles, the stage ring sized for hi + lo areas."""
    from paper_2006_05664_b200.mapping import FAMILY_TF32X3, SMEM_LIMIT

    spec = MatMulSpec(512, 1024, 1024)
    sp = gpu_operator_space(spec, "tf32x3")
    assert sp.names == gpu_operator_space(spec).names
    m = config_to_knobs(spec, sp, ((4, 2, 4, 4), (16, 1, 8, 8), (1, 32, 32), 8), "tf32x3")
    assert m.valid and m.family == FAMILY_TF32X3
    k = m.knobs
    assert (k.bm, k.bn, k.bk, k.cta_group, k.cluster) == (128, 64, 32, 1, 1)
    assert k.stages == 4 and k.smem_bytes() <= SMEM_LIMIT      # 8 wanted, 4 fit
    # an even row vthread split stays on one CTA (two M=128 atoms)
    m2 = config_to_knobs(spec, sp, ((2, 2, 8, 8), (16, 1, 8, 8), (1, 32, 32), 2), "tf32x3")
    assert m2.valid and m2.knobs.bm == 256 and m2.knobs.cta_group == 1
    # BK 4 fp32 is not a K stage
    m3 = config_to_knobs(spec, sp, ((4, 2, 4, 4), (16, 1, 8, 8), (1, 256, 4), 2), "tf32x3")
    assert not m3.valid
    with pytest.raises(TypeError):
        gpu_operator_space(parse_operator("conv2d:32,64,56,56,64,3,3,1,1"), "tf32x3")


def test_every_valid_mapping_is_prebuilt():
    """Uniform samples that map must land in the enumerated (prebuilt) family."""
    for op in ("matmul:1024,1024,1024", "batchmatmul:960,128,64,128",
               "conv2d:32,64,56,56,64,3,3,1,1", "conv2d:512,3,227,227,64,11,11,4,0",
               "conv2d:512,64,27,27,192,5,5,1,2"):
        spec = parse_operator(op)
        sp = gpu_operator_space(spec)
        fam = {(f, b, tuple(k[:4]) + tuple(k[5:])) for f, b, k in family_instances(spec)}
        # CTA pairs: MatMul 256-row tiles, conv 256-pixel tiles with an even
        # ho[1] (BMM1 has 128 rows; 55 and 27 output rows have no factor 2)
        assert any(k[9] == 2 for _, _, k in family_instances(spec)) == (
            op.startswith("matmul") or op.startswith("conv2d:32"))
        rng = np.random.default_rng(0)
        hits = 0
        for _ in range(4000):
            m = config_to_knobs(spec, sp, sp.sample_uniform(rng))
            if m.valid:
                hits += 1
                k = m.knobs.as_tuple()
                assert (m.family, m.batched, tuple(k[:4]) + tuple(k[5:])) in fam, (op, k)
        assert hits > 0


def test_every_valid_tf32x3_mapping_is_prebuilt():
    spec = parse_operator("matmul:512,1024,1024")
    sp = gpu_operator_space(spec, "tf32x3")
    fam = {(f, b, tuple(k[:4]) + tuple(k[5:])) for f, b, k in family_instances(spec, "tf32x3")}
    rng = np.random.default_rng(0)
    hits = 0
    for _ in range(3000):
        m = config_to_knobs(spec, sp, sp.sample_uniform(rng), "tf32x3")
        if m.valid:
            hits += 1
            k = m.knobs.as_tuple()
            assert (m.family, m.batched, tuple(k[:4]) + tuple(k[5:])) in fam, k
    assert hits > 0


def test_valid_fractions_recorded():
    spec = MatMulSpec(1024, 1024, 1024)
    f = valid_fraction(spec, gpu_operator_space(spec), samples=4000)
    assert 0.02 < f < 0.2


def test_opevo_runs_on_gpu_space_with_surrogate():
    """The engine drives the extended space; a surrogate stands in for the GPU."""
    spec = MatMulSpec(1024, 1024, 1024)
    sp = gpu_operator_space(spec)

    def surrogate(cfg):
        m = config_to_knobs(spec, sp, cfg)
        if not m.valid:
            return 0.0
        k = m.knobs
        return 100.0 * k.bn * k.bm / (k.bn + k.bm) / (1 + abs(k.stages - 4)) / k.split ** 0.1

    best, recs = run(sp, EngineConfig(seed=0, budget=200), surrogate)
    assert best.fitness > 0 and len(recs) == 200
