"""B200-native OpEvo: topology-aware evolutionary tuning of sm_100a kernels.

The host tuner keeps the reference's API (``topotune``, reference package
``pkg/src/topotune``): search spaces, the q-random-walk mutation,
recombination and the ask/tell loop.  The evaluator is replaced by the C-ABI
library ``libopevo.so`` (``csrc/``), which JIT-compiles, launches, verifies and
CUDA-event-times hand-written tcgen05/TMA kernels on B200.

GPU symbols (``make_gpu_objective``, ``GpuEvaluator``, ``TrialScheduler``) are
importable lazily so that the CPU-only parts load without a GPU.
"""

from .engine import (
    Archive,
    AskResult,
    EngineConfig,
    FatalEvaluationError,
    OpEvo,
    ProtocolError,
    evaluate_batch,
    mutate,
    recombine,
    run,
)
from .external import EvaluatorSpawnError, ExternalEvaluator
from .logs import Individual, TrialRecord, TrialRecorder, read_trial_log, write_trial_log
from .operators import (
    DEFAULT_COST_PARAMS,
    DESK_BATCHMATMUL,
    DESK_CONV2D,
    DESK_MATMUL,
    GOLDEN_OPTIMA,
    BatchMatMulSpec,
    Conv2dSpec,
    CostModelParams,
    MatMulSpec,
    batchmatmul_space,
    conv2d_space,
    enumerate_optimum,
    make_objective,
    matmul_space,
    operator_space,
    parse_operator,
    resource_usage,
    synthetic_cost,
)
from .reporting import (
    curve_rows,
    summarize,
    trials_to_fraction,
    tuning_report,
    wallclock_to_fraction,
)
from .spaces import (
    Categorical,
    Discrete,
    Factorization,
    ParameterSpace,
    Permutation,
    SearchSpace,
    TopologyGraph,
    build_graph,
    is_connected,
    sample_unvisited,
)
from .walk import column_sum_deviation, sample_walk, transition_matrix, walk_distribution

__version__ = "0.1.0"

_LAZY = {
    "make_gpu_objective": "evaluator",
    "GpuEvaluator": "evaluator",
    "TrialScheduler": "scheduler",
    "gpu_operator_space": "mapping",
    "config_to_knobs": "mapping",
}


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib

    return getattr(importlib.import_module(f".{mod}", __name__), name)
