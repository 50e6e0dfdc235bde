"""B200 evaluator speaking the reference's subprocess protocol.

``ExternalEvaluator`` (reference ``pkg/src/topotune/external.py:29-75``) runs one
process per configuration: ``{"params": {name: value}}`` on stdin, one
non-negative number on stdout, nonzero exit = invalid.  This program makes
the *unmodified* reference CLI drive B200 trials::

    topotune tune --space b200_matmul_1024.json --algo opevo --budget 500 \\
        --objective-cmd "python -m paper_2006_05664_b200.opevo_eval \\
                         --operator matmul:1024,1024,1024"

(write the space file with ``--dump-space``).  It prints measured TFLOP/s
for a verified kernel, ``0`` for an infeasible configuration or a wrong
result, and exits 1 on a device fault.
"""

from __future__ import annotations

import argparse
import json
import sys


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="opevo-eval")
    ap.add_argument("--operator", required=True, help="e.g. matmul:1024,1024,1024")
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--dtype", default="bf16", choices=("bf16", "f32", "tf32x3"),
                    help="f32: the SIMT family; tf32x3: fp32 on the tensor cores")
    ap.add_argument("--dump-space", action="store_true",
                    help="print the B200 search space (reference JSON format) and exit")
    args = ap.parse_args(argv)

    from .mapping import gpu_operator_space
    from .operators import parse_operator

    spec = parse_operator(args.operator)
    space = gpu_operator_space(spec, args.dtype)
    if args.dump_space:
        print(json.dumps(space.to_json()))
        return 0
    try:
        msg = json.loads(sys.stdin.readline())
        config = space.config_from_json(msg["params"])
    except (ValueError, KeyError, TypeError) as err:
        print(f"bad request: {err}", file=sys.stderr)
        return 2

    from .engine import FatalEvaluationError
    from .evaluator import DTYPES, EvalSettings, GpuEvaluator

    try:
        ev = GpuEvaluator(spec, space, args.device, EvalSettings(reps=args.reps, dtype=DTYPES[args.dtype]))
        info = ev.evaluate_infos([config])[0]
        ev.close()
    except FatalEvaluationError as err:
        print(f"device fault: {err}", file=sys.stderr)
        return 1
    if info.status != "ok":
        print(f"{info.status}: {info.message}", file=sys.stderr)
    print(repr(info.fitness))
    return 0


if __name__ == "__main__":
    sys.exit(main())
