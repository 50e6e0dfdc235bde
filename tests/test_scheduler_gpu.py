"""Multi-process trial scheduler on the GPU, including fault isolation: a
candidate that traps poisons its worker's CUDA context; the scheduler must
score it 0, replace the worker process, and keep going."""

import os
import tempfile

import pytest

pytestmark = pytest.mark.gpu


def _batch(space, n=8, seed=3):
    import numpy as np

    from paper_2006_05664_b200.mapping import config_to_knobs
    from paper_2006_05664_b200.operators import MatMulSpec

    spec = MatMulSpec(1024, 1024, 1024)
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        c = space.sample_uniform(rng)
        if config_to_knobs(spec, space, c).valid or len(out) % 2:
            out.append(c)
    return spec, out


def test_scheduler_matches_in_process_evaluation():
    from paper_2006_05664_b200.evaluator import GpuEvaluator
    from paper_2006_05664_b200.mapping import gpu_operator_space
    from paper_2006_05664_b200.operators import MatMulSpec
    from paper_2006_05664_b200.scheduler import TrialScheduler

    space = gpu_operator_space(MatMulSpec(1024, 1024, 1024))
    spec, configs = _batch(space)
    with TrialScheduler(spec, space, devices=[0]) as sched:
        fits = sched(configs)
        statuses = [e["status"] for e in sched.last_extras]
    ev = GpuEvaluator(spec, space, 0)
    try:
        ref = ev.evaluate_infos(configs)
    finally:
        ev.close()
    assert statuses == [i.status for i in ref]
    for f, i in zip(fits, ref):
        assert (f > 0) == (i.fitness > 0)


def test_trapping_candidates_are_isolated_and_the_worker_respawned():
    from paper_2006_05664_b200.evaluator import EvalSettings
    from paper_2006_05664_b200.mapping import gpu_operator_space
    from paper_2006_05664_b200.operators import MatMulSpec
    from paper_2006_05664_b200.scheduler import TrialScheduler

    space = gpu_operator_space(MatMulSpec(1024, 1024, 1024))
    spec, configs = _batch(space, n=4)
    with tempfile.TemporaryDirectory() as cache:
        old = os.environ.get("OPEVO_EXTRA_FLAGS")
        os.environ["OPEVO_EXTRA_FLAGS"] = "-DOPEVO_ABLATE=5"      # every kernel traps
        try:
            with TrialScheduler(spec, space, [0], EvalSettings(cache_dir=cache)) as sched:
                fits = sched(configs)
                extras = sched.last_extras
                assert sched.respawns >= 1
                # the scheduler still evaluates after the faults
                again = sched(configs[:1])
        finally:
            if old is None:
                os.environ.pop("OPEVO_EXTRA_FLAGS")
            else:
                os.environ["OPEVO_EXTRA_FLAGS"] = old
    assert all(f == 0.0 for f in fits)
    assert any(e["status"] == "fault" for e in extras)
    assert again == [0.0]
