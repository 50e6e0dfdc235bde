"""3xTF32 family probe: accuracy and speed of fp32 MatMul instances on the
tensor cores against the fp32 SIMT family on the same operator.
Usage: python tools/x3_probe.py matmul:512,1024,1024 128,64,32,4 ... [--simt n2,n3,...]"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2006_05664_b200 import capi  # noqa: E402
from paper_2006_05664_b200.evaluator import _op_args  # noqa: E402
from paper_2006_05664_b200.operators import parse_operator  # noqa: E402


def main():
    spec = parse_operator(sys.argv[1])
    args = sys.argv[2:]
    simt = []
    if "--simt" in args:
        i = args.index("--simt")
        simt, args = args[i + 1:], args[:i]
    dev = capi.Device(0)
    for dt, lst in ((capi.F32_TF32X3, args), (capi.F32, simt)):
        if not lst:
            continue
        op = dev.prepare(dtype=dt, seed=31, **_op_args(spec))
        ref = op.reference()
        for a in lst:
            kn = tuple(int(x) for x in a.split(","))
            t = dev.trial(op, kn, warmup=3, reps=20, tol=1.0)
            if not t.ok:
                print("x3" if dt == capi.F32_TF32X3 else "simt", kn, "FAILED", t.message)
                continue
            out = op.output()
            rel = float(np.max(np.abs(out - ref)) / np.max(np.abs(ref)))
            k = dev.kernel(op, kn)
            us = [k.time(warmup=3, reps=50, flush_l2=m) * 1e3 for m in (0, 2)]
            k.close()
            print(f"{'x3' if dt == capi.F32_TF32X3 else 'simt':4s} {kn} rel_err {rel:.2e} "
                  f"graph {us[0]:8.2f}us {spec.flops() / us[0] / 1e6:7.1f}TF | stream {us[1]:8.2f}us "
                  f"{spec.flops() / us[1] / 1e6:7.1f}TF", flush=True)
        op.close()


if __name__ == "__main__":
    main()
