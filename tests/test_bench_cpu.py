"""CPU checks of bench.py's roofline bookkeeping (no GPU): the algorithmic
bytes / FLOPs SURVEY.md §8d names, the bound chosen per operator, the dtype
ceilings, and the ncu-traffic lookup keyed by operator."""

import bench
from paper_2006_05664_b200 import parse_operator


def test_algorithmic_bytes_match_survey():
    # cfg2 6.29 MB, cfg3 62.9 MB, cfg4 25.76 MB, cfg5 100.7 MB (bf16)
    cases = {"matmul:1024,1024,1024": 6.29e6, "batchmatmul:960,128,64,128": 62.9e6,
             "conv2d:32,64,56,56,64,3,3,1,1": 25.76e6, "matmul:4096,4096,4096": 100.7e6}
    for op, want in cases.items():
        got = bench.algo_bytes(parse_operator(op), 2)
        assert abs(got - want) / want < 0.005, (op, got)
    assert bench.algo_bytes(parse_operator("matmul:512,1024,1024"), 4) == 8388608


def test_bound_follows_the_ridge():
    pk = {"tflops": 1628.2, "hbm_gbs": 6556.8}
    ridge = pk["tflops"] * 1e3 / pk["hbm_gbs"]              # ~248 flop/byte
    ai = {op: parse_operator(op).flops() / bench.algo_bytes(parse_operator(op), 2)
          for op in ("matmul:1024,1024,1024", "batchmatmul:960,128,64,128")}
    assert ai["matmul:1024,1024,1024"] > ridge > ai["batchmatmul:960,128,64,128"]


def test_dtype_ceilings():
    pk = {"tflops": 1628.2, "hbm_gbs": 6556.8, "source": "measured"}
    assert bench._dtype_peak("bf16", pk) == 1628.2
    assert abs(bench._dtype_peak("tf32x3", pk) - 1628.2 / 6) < 1e-9
    assert bench._dtype_peak("f32", pk) == bench.FP32_PEAK
    assert "3xTF32" in bench._dtype_peak_source("tf32x3", pk)


def test_ncu_traffic_is_keyed_by_operator():
    kn = (128, 64, 128, 4, 1, 1, 1, 1, 1, 1, 0, 0, 1)
    assert bench._ncu_traffic("matmul:1024,1024,1024", kn) is not None
    assert bench._ncu_traffic("matmul:2048,2048,2048", kn) is None


def test_ncu_traffic_accepts_the_14_slot_knobs():
    # bench lines carry 14 knobs since the conv `line` slot (ABI 6); a capture
    # keyed by the 13-slot tuple is the same kernel when line = 0
    kn = (128, 64, 128, 4, 1, 1, 1, 1, 1, 1, 0, 0, 1, 0)
    assert bench._ncu_traffic("matmul:1024,1024,1024", kn) is not None
    assert bench._ncu_traffic("matmul:1024,1024,1024", kn[:13] + (16,)) is None


def test_bench_compiles_without_warnings():
    # a SyntaxWarning here (e.g. two adjacent string literals read as a call)
    # is a TypeError at the end of a GPU run
    import os
    import warnings

    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "bench.py")
    with open(path) as fh:
        src = fh.read()
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        compile(src, path, "exec")


def test_fitness_timing_names_the_mode():
    import types

    from paper_2006_05664_b200.evaluator import EvalSettings

    s = EvalSettings()
    cold = bench.fitness_timing(types.SimpleNamespace(l2="cold", timing="stream"), s)
    warm = bench.fitness_timing(types.SimpleNamespace(l2="warm", timing="stream"), s)
    graph = bench.fitness_timing(types.SimpleNamespace(l2="warm", timing="graph"), s)
    assert "read pass" in cold and "gate" in warm and "CUDA graph" in graph
