"""CPU-side checks of the C-ABI library: it loads without a GPU, exports every
symbol include/opevo.h declares, JIT-compiles kernel instances (NVRTC needs
no device), rejects infeasible knobs, and fails loudly (no fallback) when
asked for a device that is not there."""

import ctypes
import os
import re

import pytest

from paper_2006_05664_b200 import capi

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "opevo.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(opevo_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(capi.library_path())
    names = declared_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(capi.EXPORTS)


def test_abi_version():
    assert capi.load().opevo_abi_version() == capi.ABI_VERSION


def test_nvrtc_compiles_instances_without_gpu(tmp_path):
    cache = str(tmp_path)
    ms = capi.compile_kernel(0, (128, 64, 64, 4, 1, 1), False, False, cache)
    assert ms > 0
    assert capi.compile_kernel(0, (128, 64, 64, 4, 1, 1), False, False, cache) == 0.0  # disk hit
    capi.compile_kernel(0, (256, 128, 128, 2, 1, 2), False, False, cache)     # 2 atoms + multicast
    capi.compile_kernel(0, (128, 48, 16, 8, 1, 1), True, False, cache)        # batched, SW32
    capi.compile_kernel(1, (128, 64, 64, 4, 1, 1, 8, 8), False, False, cache)  # implicit-GEMM conv
    files = os.listdir(cache)
    assert len(files) == 4 and all(f.endswith(".cubin") for f in files)


def test_conv_variants_compile_without_gpu(tmp_path):
    """The weight-resident (knob 11) and 256-pixel conv variants are distinct
    compile keys and build with NVRTC; the resident flag only applies to
    un-split, 128-byte-swizzle instances."""
    cache = str(tmp_path)
    capi.compile_kernel(1, (256, 64, 64, 3, 1, 1, 8, 8, 1, 1, 0, 1), False, False, cache)
    capi.compile_kernel(1, (256, 64, 64, 4, 1, 1, 8, 8), False, False, cache)
    k0 = capi.kernel_key(1, (128, 64, 64, 4, 1, 1, 8, 8), False, False)
    k1 = capi.kernel_key(1, (128, 64, 64, 4, 1, 1, 8, 8, 1, 1, 0, 1), False, False)
    k2 = capi.kernel_key(1, (128, 64, 32, 4, 1, 1, 8, 8, 1, 1, 0, 1), False, False)   # SW64: not resident
    k3 = capi.kernel_key(1, (128, 64, 32, 4, 1, 1, 8, 8), False, False)
    assert k0 != k1 and "_r_" in k1 and k2 == k3


def test_tf32x3_family_compiles_without_gpu(tmp_path):
    """Family 3 (fp32 on tcgen05, three kind::tf32 MMAs per K step): BK is in
    fp32 elements at the ABI, distinct keys from the bf16 family, and the
    bf16-only knobs (CTA pair, multicast) are rejected before NVRTC."""
    cache = str(tmp_path)
    assert capi.compile_kernel(3, (128, 64, 32, 4), False, True, cache) > 0
    capi.compile_kernel(3, (128, 64, 8, 8), True, True, cache)              # batched, SW32
    k3 = capi.kernel_key(3, (128, 64, 32, 4), False, True)
    k0 = capi.kernel_key(0, (128, 64, 64, 4), False, True)
    assert k3.startswith("f3_") and k3 != k0
    assert "_k64_" in k3          # 32 fp32 = 64 bf16 units inside the library
    for bad in [(256, 64, 32, 2, 1, 1, 1, 1, 1, 2), (128, 64, 32, 2, 1, 2),
                (128, 64, 12, 4)]:
        with pytest.raises(capi.OpevoError) as e:
            capi.compile_kernel(3, bad, False, True, cache)
        assert e.value.status == capi.INVALID_CONFIG


def test_split_is_a_launch_argument_unless_reduced_in_dsmem():
    k1 = capi.kernel_key(0, (128, 64, 64, 4, 1, 1), False, False)
    k16 = capi.kernel_key(0, (128, 64, 64, 4, 16, 1), False, False)   # global reduction
    k3 = capi.kernel_key(0, (128, 64, 64, 5, 1, 1), False, False)
    assert k1 == k16 != k3
    k2 = capi.kernel_key(0, (128, 64, 64, 4, 2, 1), False, False)     # DSMEM cluster of 2
    k8 = capi.kernel_key(0, (128, 64, 64, 4, 8, 1), False, False)
    assert len({k1, k2, k8}) == 3


@pytest.mark.parametrize("knobs", [(64, 64, 64, 4), (96, 64, 64, 4), (128, 8, 64, 4),
                                   (128, 272, 64, 4), (128, 64, 48, 4), (128, 64, 64, 40),
                                   (256, 256, 256, 2), (128, 64, 64, 4, 1, 3),
                                   (256, 512, 64, 1)])
def test_infeasible_knobs_rejected_before_compile(knobs, tmp_path):
    with pytest.raises(capi.OpevoError) as err:
        capi.compile_kernel(0, knobs, False, False, str(tmp_path))
    assert err.value.status == capi.INVALID_CONFIG
    assert os.listdir(tmp_path) == []


def test_no_device_fails_loudly():
    if os.path.exists("/dev/nvidia0"):
        pytest.skip("a GPU is present")
    with pytest.raises(capi.OpevoError) as err:
        capi.Device(0)
    assert err.value.status == capi.ERR_NO_DEVICE


def test_gpu_evaluator_raises_fatal_without_device():
    if os.path.exists("/dev/nvidia0"):
        pytest.skip("a GPU is present")
    from paper_2006_05664_b200 import FatalEvaluationError, MatMulSpec
    from paper_2006_05664_b200.evaluator import GpuEvaluator

    with pytest.raises(FatalEvaluationError):
        GpuEvaluator(MatMulSpec(256, 256, 256))


def test_narrow_epilogue_rule_matches_the_mapping():
    """The two-CTAs-per-SM rule (32-column epilogue staging, key suffix
    ``_e32``) is decided the same way by the library and by mapping.py, over
    every instance of the conv cfg4, BMM1 and 1024^3 families."""
    from paper_2006_05664_b200.mapping import Knobs
    from paper_2006_05664_b200.operators import parse_operator
    from paper_2006_05664_b200.prebuild import family_instances

    seen = 0
    for opid in ("conv2d:32,64,56,56,64,3,3,1,1", "batchmatmul:960,128,64,128", "matmul:1024,1024,1024"):
        for fam, batched, kn in family_instances(parse_operator(opid)):
            narrow = Knobs(*kn, family=fam, batched=int(batched)).narrow_epi()
            assert ("_e32" in capi.kernel_key(fam, kn, batched, False)) == narrow, kn
            seen += narrow
    assert seen > 100
    # a 2-stage halo conv tile: 114 KB with 64-column staging, 98 KB with 32
    halo2 = Knobs(128, 64, 64, 2, 1, 1, 1, 14, family=1)
    assert halo2.narrow_epi() and halo2.smem_bytes() == 80 * 1024 + 16 * 1024 + 1280
    assert not Knobs(128, 64, 64, 3, 1, 1, 1, 14, family=1).narrow_epi()


def test_512_row_pairs_only_for_halo_conv(tmp_path):
    """BM = 512 (256 rows per CTA of a pair) exists only as a halo-line conv
    CTA pair; the library rejects it for GEMM tiles, single CTAs and dense
    conv tiles before NVRTC, and compiles the halo pair."""
    cache = str(tmp_path)
    assert capi.compile_kernel(1, (512, 64, 64, 3, 1, 1, 4, 14, 1, 2, 0, 0, 1, 0), False, False, cache) > 0
    for fam, bad in [(0, (512, 64, 64, 3, 1, 1, 1, 1, 1, 2)), (1, (512, 64, 64, 3, 1, 1, 4, 14, 1, 1)),
                     (1, (512, 64, 64, 3, 1, 1, 8, 8, 1, 2))]:
        with pytest.raises(capi.OpevoError) as e:
            capi.compile_kernel(fam, bad, False, False, cache)
        assert e.value.status == capi.INVALID_CONFIG, bad
