"""Per-CTA phase breakdown of one kernel instance (debug build with
-DOPEVO_TRACE=1).  Usage: python tools/trace_kernel.py matmul:1024,1024,1024 128,64,256,2,1,1"""
import os
import sys

os.environ["OPEVO_EXTRA_FLAGS"] = "-DOPEVO_TRACE=1"
sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2006_05664_b200 import capi  # noqa: E402
from paper_2006_05664_b200.evaluator import _op_args  # noqa: E402
from paper_2006_05664_b200.operators import parse_operator  # noqa: E402

PHASES = [("launch skew", None, 1), ("setup", 1, 2), ("pdl wait", 2, 9), ("first TMA issue", 9, 3),
          ("first stage landed", 3, 4), ("mainloop", 4, 5), ("accum->epi", 5, 6),
          ("epilogue", 6, 7), ("exit sync", 7, 8), ("CTA total", 1, 8)]


def main():
    spec = parse_operator(sys.argv[1])
    knobs = tuple(int(x) for x in sys.argv[2].split(","))
    dev = capi.Device(0, "/tmp/opevo_trace_cache")
    op = dev.prepare(**_op_args(spec))
    k = dev.kernel(op, knobs)
    ctas = k.info.grid_ctas
    for _ in range(5):              # warm L2 and the instruction cache
        k.trace(ctas)
    tr = k.trace(ctas).astype(np.int64)
    t0 = tr[:, 1].min()
    print(f"{spec.id()} knobs={knobs} ctas={ctas} distinct SMs={len(set(tr[:, 0]))}")
    for name, a, b in PHASES:
        d = (tr[:, b] - (t0 if a is None else tr[:, a])) / 1e3
        print(f"  {name:20s} min {d.min():7.2f}  med {np.median(d):7.2f}  max {d.max():7.2f} us")
    print(f"  kernel span (first entry -> last exit): {(tr[:, 8].max() - t0) / 1e3:.2f} us")
    k.close()


if __name__ == "__main__":
    main()
