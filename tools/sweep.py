"""Time a list of knob tuples on one operator (verified trials).
Usage: python tools/sweep.py OP "bm,bn,bk,st,split,cl,th,tw,acc" ...  (or --grid)"""
import itertools
import sys

sys.path.insert(0, ".")
from paper_2006_05664_b200 import capi  # noqa: E402
from paper_2006_05664_b200.evaluator import _op_args  # noqa: E402
from paper_2006_05664_b200.operators import parse_operator  # noqa: E402


def main():
    spec = parse_operator(sys.argv[1])
    dev = capi.Device(0)
    op = dev.prepare(**_op_args(spec))
    if sys.argv[2] == "--grid":
        grid = [tuple(int(x) for x in g.split(",")) for g in sys.argv[3].split(";")]
        cases = list(itertools.product(*grid))
    else:
        cases = [tuple(int(x) for x in a.split(",")) for a in sys.argv[2:]]
    res = []
    for kn in cases:
        t = dev.trial(op, kn, warmup=5, reps=50)
        if t.status == capi.INVALID_CONFIG:
            continue
        res.append((t.tflops, kn, t.status, t.message[:60]))
    res.sort(reverse=True)
    for r in res[:40]:
        print("%7.1f TFLOP/s  %s  st=%d %s" % r)
    print("non-ok:", [r for r in res if r[2] != 0][:5])


if __name__ == "__main__":
    main()
