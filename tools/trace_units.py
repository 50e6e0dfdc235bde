"""Per-unit MMA -> epilogue handshake of a persistent instance (debug build
with -DOPEVO_TRACE=2): for the first five units of every CTA, when the MMA
warp issued the unit's accumulator commit, when the epilogue saw it, and
when the epilogue finished the unit (medians over CTAs, us from CTA entry
of the earliest CTA).  Ablation flags may be added through OPEVO_ABLATE_FLAG.
Usage: python tools/trace_units.py batchmatmul:960,128,64,128 128,64,64,6,1,1"""
import os
import sys

MODE = int(os.environ.get("OPEVO_TRACE_MODE", "2"))
os.environ["OPEVO_EXTRA_FLAGS"] = (f"-DOPEVO_TRACE={MODE} " + os.environ.get("OPEVO_ABLATE_FLAG", "")).strip()
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
    if MODE == 3:
        # MMA warp per unit: accumulator free (start), first stage ready, commit issued
        print("  unit   start   first-stage-ready   commit-issued   (us; wait-for-data, issue, gap-to-next-start)")
        prev = None
        for u in range(5):
            a, b, c = tr[:, 1 + 3 * u], tr[:, 2 + 3 * u], tr[:, 3 + 3 * u]
            ok = (a > 0) & (b > 0) & (c > 0)
            if not ok.any():
                break
            t0 = tr[ok, 1].min()
            ma, mb, mc = (np.median(x[ok] - t0) / 1e3 for x in (a, b, c))
            gap = "" if prev is None else f", gap {ma - prev:.2f}"
            print(f"  {u:4d}   {ma:5.2f}   {mb:17.2f}   {mc:13.2f}   (data {mb - ma:.2f}, issue {mc - mb:.2f}{gap})")
            prev = mc
        k.close()
        return
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
