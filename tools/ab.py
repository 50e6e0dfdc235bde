"""Interleaved A/B timing of kernel instances on one operator (same process,
rounds alternate between candidates so clock/thermal drift hits all equally).
Usage: python tools/ab.py OP ROUNDS knobsA knobsB ..."""
import statistics
import subprocess
import sys

sys.path.insert(0, ".")
from paper_2006_05664_b200 import capi  # noqa: E402
from paper_2006_05664_b200.evaluator import _op_args  # noqa: E402
from paper_2006_05664_b200.operators import parse_operator  # noqa: E402


def sm_clock():
    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=5).stdout.strip()
        return out
    except Exception:  # noqa: BLE001
        return "?"


def main():
    spec = parse_operator(sys.argv[1])
    rounds = int(sys.argv[2])
    cands = [tuple(int(x) for x in a.split(",")) for a in sys.argv[3:]]
    dev = capi.Device(0)
    op = dev.prepare(**_op_args(spec))
    ks, ok = [], []
    for c in cands:
        try:
            k = dev.kernel(op, c)
            err = k.check()
        except capi.OpevoError as e:
            print(f"  {str(c):48s} skipped: {e}")
            continue
        print(f"  {str(c):48s} rel err {err:.2e}")
        ks.append(k)
        ok.append(c)
    cands = ok
    res = {c: [] for c in cands}
    for _ in range(rounds):
        for c, k in zip(cands, ks):
            ms = k.time(warmup=3, reps=30)
            res[c].append(spec.flops() / ms / 1e9)
    print(f"{spec.id()}  rounds={rounds}  clock/power after: {sm_clock()}")
    for c in cands:
        v = res[c]
        print(f"  {str(c):48s} median {statistics.median(v):7.1f}  min {min(v):7.1f}  max {max(v):7.1f} TFLOP/s")


if __name__ == "__main__":
    main()
