"""Same instances, different timing modes (graph = 0, gated stream = 2),
interleaved rounds.  Usage: python tools/timing_mode_ab.py OP REPS knobs..."""
import statistics
import sys

sys.path.insert(0, ".")
from paper_2006_05664_b200 import capi  # noqa: E402
from paper_2006_05664_b200.evaluator import _op_args  # noqa: E402
from paper_2006_05664_b200.operators import parse_operator  # noqa: E402


def main():
    spec = parse_operator(sys.argv[1])
    reps = int(sys.argv[2])
    cands = [tuple(int(x) for x in a.split(",")) for a in sys.argv[3:]]
    dev = capi.Device(0)
    op = dev.prepare(**_op_args(spec))
    ks = [dev.kernel(op, c) for c in cands]
    res = {(c, m): [] for c in cands for m in (0, 2)}
    for _ in range(5):
        for c, k in zip(cands, ks):
            for m in (0, 2):
                ms = k.time(warmup=3, reps=reps, flush_l2=m)
                res[(c, m)].append(spec.flops() / ms / 1e9)
    print(f"{spec.id()} reps={reps}")
    for c in cands:
        g, s = res[(c, 0)], res[(c, 2)]
        print(f"  {str(c):44s} graph median {statistics.median(g):7.1f} [{min(g):7.1f},{max(g):7.1f}]  "
              f"stream median {statistics.median(s):7.1f} [{min(s):7.1f},{max(s):7.1f}] TFLOP/s")


if __name__ == "__main__":
    main()
