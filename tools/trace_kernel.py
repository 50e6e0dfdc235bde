"""Per-CTA phase breakdown of one kernel instance (debug build with
-DOPEVO_TRACE=1).  Usage: python tools/trace_kernel.py matmul:1024,1024,1024 128,64,256,2,1,1 [launches]

With launches > 1 the launches run back to back (PDL, as in the fitness
timing) and a steady-state timeline is printed: per launch, the first CTA
entry, median post-PDL-wait, first MMA, mainloop end and last exit, relative
to the first launch's first entry."""
import os
import sys

os.environ["OPEVO_EXTRA_FLAGS"] = "-DOPEVO_TRACE=1"
sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2006_05664_b200 import capi  # noqa: E402
from paper_2006_05664_b200.evaluator import _op_args  # noqa: E402
from paper_2006_05664_b200.operators import parse_operator  # noqa: E402

PHASES = [("launch skew", None, 1), ("setup", 1, 2), ("pdl wait", 2, 9),
          ("  wait->empty ok", 9, 10), ("  ->expect_tx", 10, 11), ("  ->TMAs issued", 11, 3),
          ("  epi: first LDTM", 6, 12), ("  epi: first stores", 12, 13), ("first TMA issue", 9, 3),
          ("first stage landed", 3, 4), ("mainloop", 4, 5), ("accum->epi", 5, 6),
          ("epilogue", 6, 7), ("exit sync", 7, 8), ("CTA total", 1, 8),
          # DSMEM split-K reduction (OPEVO_SPLIT_CLUSTER): stage own partial,
          # cluster sync, peers' blocks landed, sum + store; then exit sync
          ("dsmem: stage own", 6, 12), ("dsmem: cluster sync", 12, 13), ("dsmem: recv wait", 13, 14),
          ("dsmem: sum+store", 14, 7), ("final cluster sync", 8, 15)]


def main():
    spec = parse_operator(sys.argv[1])
    knobs = tuple(int(x) for x in sys.argv[2].split(","))
    nl = int(sys.argv[3]) if len(sys.argv) > 3 else 1
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
        # stamps a CTA never writes (e.g. MMA stamps of a CTA-pair follower) are 0
        ok = (tr[:, b] != 0) & ((tr[:, a] != 0) if a is not None else True)
        if not ok.any():
            print(f"  {name:20s} (no stamps)")
            continue
        d = (tr[ok, b] - (t0 if a is None else tr[ok, a])) / 1e3
        print(f"  {name:20s} min {d.min():7.2f}  med {np.median(d):7.2f}  max {d.max():7.2f} us")
    print(f"  kernel span (first entry -> last exit): {(tr[:, 8].max() - t0) / 1e3:.2f} us")
    if nl > 1:
        for _ in range(3):
            k.trace(ctas, nl)
        tl = k.trace(ctas, nl).astype(np.int64)
        z = tl[0, :, 1].min()
        print(f"  back-to-back x{nl} (us from launch 0 first entry):")
        print("    launch  first-entry  med-entry  med-post-wait  med-first-MMA  med-MMA-done  "
              "med-epi-done  last-exit")
        def med(col):
            v = col[col != 0]
            return np.median((v - z) / 1e3) if v.size else float("nan")

        for i in range(nl):
            t = (tl[i] - z) / 1e3
            print(f"    {i:6d}  {t[:, 1].min():11.2f}  {med(tl[i][:, 1]):9.2f}  {med(tl[i][:, 9]):13.2f}"
                  f"  {med(tl[i][:, 4]):13.2f}  {med(tl[i][:, 5]):12.2f}  {med(tl[i][:, 7]):12.2f}"
                  f"  {t[:, 8].max():9.2f}")
        span = (tl[-1, :, 8].max() - tl[0, :, 1].min()) / 1e3
        print(f"  steady state: {span / nl:.2f} us per launch over {nl} launches")
    k.close()


if __name__ == "__main__":
    main()
