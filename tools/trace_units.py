"""Per-unit MMA -> epilogue handshake of a persistent instance (debug build
with -DOPEVO_TRACE=2): for the first five units of every CTA, when the MMA
warp issued the unit's accumulator commit, when the epilogue saw it, and
when the epilogue finished the unit (medians over CTAs, us from CTA entry
of the earliest CTA).  Ablation flags may be added through OPEVO_ABLATE_FLAG.
Usage: python tools/trace_units.py batchmatmul:960,128,64,128 128,64,64,6,1,1"""
import os
import sys

os.environ["OPEVO_EXTRA_FLAGS"] = ("-DOPEVO_TRACE=2 " + os.environ.get("OPEVO_ABLATE_FLAG", "")).strip()
sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2006_05664_b200 import capi  # noqa: E402
from paper_2006_05664_b200.evaluator import _op_args  # noqa: E402
from paper_2006_05664_b200.operators import parse_operator  # noqa: E402


def main():
    spec = parse_operator(sys.argv[1])
    knobs = tuple(int(x) for x in sys.argv[2].split(","))
    dev = capi.Device(0, "/tmp/opevo_trace_units_cache")
    op = dev.prepare(**_op_args(spec))
    k = dev.kernel(op, knobs)
    ctas = k.info.grid_ctas
    for _ in range(5):
        k.trace(ctas)
    tr = k.trace(ctas).astype(np.int64)
    print(f"{spec.id()} knobs={knobs} ctas={ctas} {os.environ['OPEVO_EXTRA_FLAGS']}")
    print("  unit   commit-issued   epilogue-saw   epilogue-done   (us, median over CTAs; "
          "saw-commit, done-saw)")
    rows = []
    for u in range(5):
        c, sw, d = tr[:, 1 + 3 * u], tr[:, 2 + 3 * u], tr[:, 3 + 3 * u]
        ok = (c > 0) & (sw > 0) & (d > 0)
        if not ok.any():
            break
        t0 = tr[ok, 1].min()
        rows.append((u, np.median(c[ok] - t0) / 1e3, np.median(sw[ok] - t0) / 1e3, np.median(d[ok] - t0) / 1e3,
                     np.median(sw[ok] - c[ok]) / 1e3, np.median(d[ok] - sw[ok]) / 1e3))
    for u, c, sw, d, l1, l2 in rows:
        print(f"  {u:4d}   {c:13.2f}   {sw:12.2f}   {d:13.2f}   ({l1:.2f}, {l2:.2f})")
    k.close()


if __name__ == "__main__":
    main()
