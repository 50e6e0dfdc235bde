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


def test_two_rank_gloo_bench_survives_a_trapping_candidate(tmp_path):
    """bench.py on two ranks (gloo exchange, both on GPU 0) with one kernel
    instance built to trap (OPEVO_FAULT_KNOBS, a sticky fault that poisons
    the evaluating rank's CUDA context): the run completes, the faulting
    trial scores 0 with status "fault", and the faulted rank carries on in
    a worker process."""
    import json
    import socket
    import subprocess
    import sys

    from paper_2006_05664_b200 import EngineConfig
    from paper_2006_05664_b200.mapping import config_to_knobs, gpu_operator_space
    from paper_2006_05664_b200.native import NativeOpEvo
    from paper_2006_05664_b200.operators import MatMulSpec

    spec = MatMulSpec(1024, 1024, 1024)
    space = gpu_operator_space(spec)
    # a seed whose first (uniform, fitness-independent) batch holds a valid
    # configuration: its instance is the one built to trap
    for seed in range(200):
        first = NativeOpEvo(space, EngineConfig(seed=seed, budget=64)).ask().configs
        valid = [config_to_knobs(spec, space, c) for c in first]
        valid = [m for m in valid if m.valid]
        if valid:
            break
    knobs = ",".join(map(str, valid[0].knobs.as_tuple()))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, OPEVO_DIST_BACKEND="gloo", OPEVO_FAULT_KNOBS=knobs)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", "bench.py", "--gpus", "2",
           "--steps", "6", "--warmup", "3", "--budget", "96", "--seed", str(seed), "--no-e2e",
           "--no-cpu", "--no-cold"]
    out = subprocess.run(cmd, cwd=repo, env=env, capture_output=True, text=True, timeout=900)
    if out.returncode != 0:
        pytest.fail("bench failed:\n" + out.stdout[-2000:] + "\n" + out.stderr[-6000:])
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["faulted_trials"] >= 1
    assert line["trials_total"] == 96 and line["value"] > 0
