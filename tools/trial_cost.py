"""Where a trial's wall time goes: kernel_get (disk cache read + module load +
tensor maps), check (poisoned launch + compare), time (warm-up + estimate +
graph of R launches).  Usage: python tools/trial_cost.py [op] [n]"""
import statistics
import sys
import time

sys.path.insert(0, ".")
from paper_2006_05664_b200 import capi  # noqa: E402
from paper_2006_05664_b200.evaluator import _op_args  # noqa: E402
from paper_2006_05664_b200.operators import parse_operator  # noqa: E402


def main():
    op_id = sys.argv[1] if len(sys.argv) > 1 else "matmul:1024,1024,1024"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    spec = parse_operator(op_id)
    dev = capi.Device(0)
    op = dev.prepare(**_op_args(spec))
    cands = []
    for bn in (64, 128, 256, 32, 16, 48, 96, 192):
        for bk in (64, 128, 32):
            for st in (2, 3, 4, 6):
                cands.append((128, bn, bk, st, 1, 1))
    cands = cands[:n]
    rows = {"get": [], "check": [], "time": [], "trial": [], "get_warm": []}
    for kn in cands:
        t0 = time.perf_counter()
        try:
            k = dev.kernel(op, kn)
        except capi.OpevoError:
            continue
        t1 = time.perf_counter()
        k.check()
        t2 = time.perf_counter()
        k.time(warmup=3, reps=20)
        t3 = time.perf_counter()
        k.close()
        t4 = time.perf_counter()
        k2 = dev.kernel(op, kn)
        t5 = time.perf_counter()
        k2.close()
        tr0 = time.perf_counter()
        dev.trial(op, kn)
        tr1 = time.perf_counter()
        rows["get"].append(t1 - t0)
        rows["check"].append(t2 - t1)
        rows["time"].append(t3 - t2)
        rows["get_warm"].append(t5 - t4)
        rows["trial"].append(tr1 - tr0)
    valid = [kn for kn in cands]
    bt = []
    for lo in range(0, len(valid), 8):
        t0 = time.perf_counter()
        res = dev.trial_batch(op, valid[lo:lo + 8])
        bt.append((time.perf_counter() - t0) / max(1, sum(r.ok for r in res)))
    rows["batch_per_ok_trial"] = bt
    for name, v in rows.items():
        print(f"{name:9s} n={len(v)} median {1e3 * statistics.median(v):.3f} ms  "
              f"mean {1e3 * statistics.mean(v):.3f} ms  max {1e3 * max(v):.3f} ms")


if __name__ == "__main__":
    main()
