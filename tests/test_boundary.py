"""The reference-facing boundaries beside the C ABI.

1. The subprocess protocol (reference ``external.py:29-75``): the B200
   evaluator program ``opevo_eval`` speaks it, its ``--dump-space`` output is a
   space file the reference loads (``SearchSpace.from_json``,
   ``spaces.py:411-434``) and its ``tune --space --objective-cmd`` path
   (``cli.py:76-103``) drives, and both the reference's and this package's
   ``ExternalEvaluator`` map every failure mode to fitness 0.
2. Reporting (reference ``reporting.py:33-118``): ``summarize``,
   ``curve_rows`` and the two CSV writers of this package produce
   byte-identical files to the reference's on the same trial logs.
"""

import gzip
import json
import os
import subprocess
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
OP = "matmul:1024,1024,1024"


def _eval_cmd(*extra: str) -> str:
    return " ".join([sys.executable, "-m", "paper_2006_05664_b200.opevo_eval", "--operator", OP,
                     *extra])


def _run_eval(stdin: str, *extra: str, timeout: float = 60.0):
    return subprocess.run([sys.executable, "-m", "paper_2006_05664_b200.opevo_eval", "--operator", OP,
                           *extra], input=stdin, capture_output=True, text=True, cwd=REPO,
                          timeout=timeout)


@pytest.fixture(scope="module")
def dumped_space():
    out = _run_eval("", "--dump-space")
    assert out.returncode == 0, out.stderr
    return json.loads(out.stdout)


def test_dump_space_is_the_gpu_space(dumped_space):
    from paper_2006_05664_b200.mapping import gpu_operator_space
    from paper_2006_05664_b200.operators import parse_operator
    from paper_2006_05664_b200.spaces import SearchSpace

    ours = gpu_operator_space(parse_operator(OP))
    assert dumped_space == ours.to_json()
    back = SearchSpace.from_json(dumped_space)
    assert back.names == ours.names and back.size() == ours.size()


def test_dump_space_loads_in_the_reference(dumped_space, reference_topotune, tmp_path):
    """The reference's own loader accepts the B200 space (the JSON format is
    the interoperability contract) and enumerates the same configurations."""
    from paper_2006_05664_b200.spaces import SearchSpace

    ref = reference_topotune.spaces.SearchSpace.from_json(dumped_space)
    ours = SearchSpace.from_json(dumped_space)
    assert list(ref.names) == list(ours.names)
    assert ref.size() == ours.size()
    rng_a, rng_b = np.random.default_rng(5), np.random.default_rng(5)
    for _ in range(50):
        ca, cb = ref.sample_uniform(rng_a), ours.sample_uniform(rng_b)
        assert ca == cb
        assert ref.config_to_json(ca) == ours.config_to_json(cb)
    path = tmp_path / "b200_space.json"
    path.write_text(json.dumps(dumped_space))
    assert reference_topotune.spaces.SearchSpace.from_file(str(path)).size() == ours.size()


@pytest.mark.parametrize("stdin", ["", "not json\n", '{"params": {"n": [1, 2]}}\n', '{"x": 1}\n'])
def test_opevo_eval_rejects_bad_requests(stdin):
    out = _run_eval(stdin)
    assert out.returncode == 2
    assert "bad request" in out.stderr


def test_opevo_eval_device_fault_exits_nonzero(dumped_space):
    """No such device: the program reports a fault (exit 1), which the
    protocol scores 0 -- on a CPU host and on a GPU box alike."""
    from paper_2006_05664_b200.spaces import SearchSpace

    space = SearchSpace.from_json(dumped_space)
    cfg = space.sample_uniform(np.random.default_rng(0))
    out = _run_eval(json.dumps({"params": space.config_to_json(cfg)}) + "\n", "--device", "97")
    assert out.returncode == 1, out.stderr
    assert "device fault" in out.stderr


@pytest.mark.parametrize("which", ["ours", "reference"])
def test_external_evaluator_failure_modes(which, dumped_space, reference_topotune, tmp_path,
                                          monkeypatch):
    """Both ExternalEvaluator implementations score every failure 0: a fault
    exit, a timeout, garbage or negative output; and a spawn failure is fatal."""
    from paper_2006_05664_b200 import external as ours_ext
    from paper_2006_05664_b200.engine import FatalEvaluationError
    from paper_2006_05664_b200.spaces import SearchSpace

    if which == "ours":
        ext, space = ours_ext, SearchSpace.from_json(dumped_space)
        fatal = FatalEvaluationError
    else:
        ext = reference_topotune.external
        space = reference_topotune.spaces.SearchSpace.from_json(dumped_space)
        fatal = reference_topotune.engine.FatalEvaluationError
    cfg = space.sample_uniform(np.random.default_rng(1))
    monkeypatch.setenv("PYTHONPATH", REPO + os.pathsep + os.environ.get("PYTHONPATH", ""))
    assert ext.ExternalEvaluator(_eval_cmd("--device", "97"), space, 60000)(cfg) == 0.0
    assert ext.ExternalEvaluator(_eval_cmd(), space, 1)(cfg) == 0.0          # 1 ms timeout
    for body in ("print('garbage')", "print(-3.5)", "print('nan')", "import sys; sys.exit(3)"):
        script = tmp_path / "child.py"
        script.write_text(f"import sys\nsys.stdin.read()\n{body}\n")
        assert ext.ExternalEvaluator(f"{sys.executable} {script}", space, 60000)(cfg) == 0.0
    script = tmp_path / "ok.py"
    script.write_text("import sys\nsys.stdin.read()\nprint('noise')\nprint(12.5)\n")
    assert ext.ExternalEvaluator(f"{sys.executable} {script}", space, 60000)(cfg) == 12.5
    with pytest.raises(fatal):
        ext.ExternalEvaluator("/nonexistent/opevo-eval", space, 1000)(cfg)


def test_reference_cli_drives_opevo_eval(dumped_space, reference_topotune, tmp_path):
    """The unmodified reference CLI (``topotune tune --space FILE
    --objective-cmd CMD``) runs a search through opevo_eval.  Here the
    command names a device that does not exist, so every trial is a fault
    scored 0 -- the point is the wiring: the space file, the request format
    and the reply parsing are the reference's own."""
    space_file = tmp_path / "b200.json"
    space_file.write_text(json.dumps(dumped_space))
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.dirname(os.path.dirname(
        reference_topotune.__file__)), REPO])
    out = subprocess.run([sys.executable, "-m", "topotune", "tune", "--space", str(space_file),
                          "--objective-cmd", _eval_cmd("--device", "97"), "--budget", "8",
                          "--seed", "3", "--out", str(tmp_path / "out")],
                         capture_output=True, text=True, cwd=str(tmp_path), env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    logs = [p for p in (tmp_path / "out").rglob("*.jsonl")]
    assert logs, list((tmp_path / "out").rglob("*"))
    recs = [json.loads(x) for x in logs[0].read_text().splitlines() if x.strip()]
    assert len(recs) == 8 and all(r["fitness"] == 0.0 for r in recs)


@pytest.mark.gpu
def test_opevo_eval_measures_on_the_gpu(dumped_space, monkeypatch):
    """On a B200: a valid configuration yields its measured TFLOP/s, an
    infeasible one 0, through this package's ExternalEvaluator."""
    from paper_2006_05664_b200.external import ExternalEvaluator
    from paper_2006_05664_b200.mapping import config_to_knobs
    from paper_2006_05664_b200.operators import parse_operator
    from paper_2006_05664_b200.spaces import SearchSpace

    space = SearchSpace.from_json(dumped_space)
    spec = parse_operator(OP)
    rng = np.random.default_rng(0)
    valid = invalid = None
    while valid is None or invalid is None:
        c = space.sample_uniform(rng)
        if config_to_knobs(spec, space, c).valid:
            valid = valid or c
        else:
            invalid = invalid or c
    monkeypatch.setenv("PYTHONPATH", REPO + os.pathsep + os.environ.get("PYTHONPATH", ""))
    ev = ExternalEvaluator(_eval_cmd(), space, 120000)
    assert ev(valid) > 0.0
    assert ev(invalid) == 0.0


# ------------------------------------------------------------------ reporting
def _reference_logs(topotune, seeds=(0, 1, 2), budget=120):
    from topotune.benchmarks import make_objective, parse_operator
    from topotune.engine import EngineConfig, run

    space, obj = make_objective(parse_operator("matmul:512,1024,1024"))
    return [run(space, EngineConfig(seed=s, budget=budget), obj)[1] for s in seeds]


def _gpu_log_records(mod):
    """The committed B200 trial log (reference schema + extras) as TrialRecords
    of package ``mod`` (extras dropped: the reference schema has none)."""
    keys = ("trial", "config", "fitness", "best_so_far", "elapsed_ms")
    with gzip.open(os.path.join(GOLDEN, "gpu_trial_log_mm1024_seed0.jsonl.gz"), "rt") as fh:
        rows = [json.loads(x) for x in fh if x.strip()]
    return [mod.TrialRecord.from_json(json.dumps({k: r[k] for k in keys})) for r in rows]


def test_reporting_csvs_byte_identical(reference_topotune, tmp_path):
    from paper_2006_05664_b200 import logs as our_logs
    from paper_2006_05664_b200 import reporting as ours
    from topotune import logs as ref_logs
    from topotune import reporting as ref

    runs = _reference_logs(reference_topotune)
    ref_runs = runs + [_gpu_log_records(ref_logs)]
    # the same logs through this package's reader
    our_runs = []
    for i, lg in enumerate(ref_runs):
        p = tmp_path / f"log{i}.jsonl"
        ref_logs.write_trial_log(str(p), lg)
        our_runs.append(our_logs.read_trial_log(str(p)))
    for a, b in zip(ref_runs, our_runs):
        assert ref.trials_to_fraction(a) == ours.trials_to_fraction(b)
    rs, os_ = ref.summarize("opevo", "mm", ref_runs), ours.summarize("opevo", "mm", our_runs)
    ref.write_summary_csv(str(tmp_path / "ref_summary.csv"), [ref.summary_row_dict(rs, space="mm")])
    ours.write_summary_csv(str(tmp_path / "our_summary.csv"), [ours.summary_row_dict(os_, space="mm")])
    ref.write_curves_csv(str(tmp_path / "ref_curves.csv"), ref.curve_rows("opevo", ref_runs, 600))
    ours.write_curves_csv(str(tmp_path / "our_curves.csv"), ours.curve_rows("opevo", our_runs, 600))
    for name in ("summary", "curves"):
        assert (tmp_path / f"ref_{name}.csv").read_bytes() == (tmp_path / f"our_{name}.csv").read_bytes()


def test_wallclock_to_fraction_is_elapsed_of_trials_to_fraction(reference_topotune):
    from paper_2006_05664_b200 import reporting as ours
    from paper_2006_05664_b200 import logs as our_logs

    recs = _gpu_log_records(our_logs)
    t = ours.trials_to_fraction(recs)
    assert ours.wallclock_to_fraction(recs) == next(r.elapsed_ms for r in recs if r.trial == t)
    assert t == reference_topotune.reporting.trials_to_fraction(_gpu_log_records(reference_topotune.logs))


def test_sweep_matches_the_reference_cli(reference_topotune, tmp_path):
    """``sweep`` (OpEvo's q / lambda grid, reference ``cli.py:237-270``) with the
    reference's synthetic evaluator: the same cell directories, the same trial
    logs (configs and fitness, trial by trial) and the same sweep_summary.csv
    apart from the wall-clock column."""
    import csv

    args = ["--q-grid", "0.25,0.75", "--lambda-grid", "4,8", "--seeds", "0,3", "--budget", "60"]
    env = dict(os.environ, PYTHONPATH=os.path.dirname(os.path.dirname(reference_topotune.__file__)))
    ref = subprocess.run([sys.executable, "-m", "topotune", "sweep", "--operator", "matmul:512,1024,1024",
                          *args, "--out", str(tmp_path / "ref")], capture_output=True, text=True, env=env,
                         timeout=300)
    assert ref.returncode == 0, ref.stderr
    ours = subprocess.run([sys.executable, "-m", "paper_2006_05664_b200", "sweep", "--operator",
                           "matmul:512,1024,1024", "--evaluator", "synthetic", *args, "--out",
                           str(tmp_path / "ours")], capture_output=True, text=True, cwd=REPO, timeout=300)
    assert ours.returncode == 0, ours.stderr
    cells = sorted(p.name for p in (tmp_path / "ref").iterdir() if p.is_dir())
    assert cells == sorted(p.name for p in (tmp_path / "ours").iterdir() if p.is_dir()) and len(cells) == 4
    for cell in cells:
        for seed in (0, 3):
            name = f"trials_opevo_seed{seed}.jsonl"
            a = [json.loads(x) for x in (tmp_path / "ref" / cell / name).read_text().splitlines()]
            b = [json.loads(x) for x in (tmp_path / "ours" / cell / name).read_text().splitlines()]
            assert [(r["config"], r["fitness"]) for r in a] == [(r["config"], r["fitness"]) for r in b]

    def rows(path):
        with open(path) as fh:
            return [{k: v for k, v in r.items() if k != "mean_elapsed_ms"} for r in csv.DictReader(fh)]

    assert rows(tmp_path / "ref" / "sweep_summary.csv") == rows(tmp_path / "ours" / "sweep_summary.csv")


def test_bench_matches_the_reference_cli(reference_topotune, tmp_path):
    """``bench`` (the reference CLI's name for comparing algorithms over seeds,
    ``cli.py:189-233``; ``compare`` here) with the reference's synthetic
    evaluator and non-default q / lambda: the same trial logs and the same
    summary.csv (apart from wall clock) and curves.csv."""
    import csv

    args = ["--algo", "opevo,random,sa,gbfs", "--seeds", "0,5", "--budget", "48", "--q", "0.3",
            "--lambda", "4"]
    env = dict(os.environ, PYTHONPATH=os.path.dirname(os.path.dirname(reference_topotune.__file__)))
    ref = subprocess.run([sys.executable, "-m", "topotune", "bench", "--operator", "matmul:512,1024,1024",
                          *args, "--out", str(tmp_path / "ref")], capture_output=True, text=True, env=env,
                         timeout=300)
    assert ref.returncode == 0, ref.stderr
    ours = subprocess.run([sys.executable, "-m", "paper_2006_05664_b200", "bench", "--operator",
                           "matmul:512,1024,1024", "--evaluator", "synthetic", *args, "--out",
                           str(tmp_path / "ours")], capture_output=True, text=True, cwd=REPO, timeout=300)
    assert ours.returncode == 0, ours.stderr
    for algo in ("opevo", "random", "sa", "gbfs"):
        for seed in (0, 5):
            name = f"trials_{algo}_seed{seed}.jsonl"
            a = [json.loads(x) for x in (tmp_path / "ref" / name).read_text().splitlines()]
            b = [json.loads(x) for x in (tmp_path / "ours" / name).read_text().splitlines()]
            assert [(r["config"], r["fitness"]) for r in a] == [(r["config"], r["fitness"]) for r in b]

    def rows(path, drop=("mean_elapsed_ms",)):
        with open(path) as fh:
            return [{k: v for k, v in r.items() if k not in drop} for r in csv.DictReader(fh)]

    assert rows(tmp_path / "ref" / "summary.csv") == rows(tmp_path / "ours" / "summary.csv")
    assert rows(tmp_path / "ref" / "curves.csv") == rows(tmp_path / "ours" / "curves.csv")
