"""Exhaustive ground truth for a search: time EVERY kernel instance the
operator's space maps to (prebuild.family_instances, the prebuilt cubins)
and print the fastest -- the optimum OpEvo should find.
Usage: python tools/sweep_family.py OP [top] [reps]"""
import sys
import time

sys.path.insert(0, ".")
from paper_2006_05664_b200 import capi  # noqa: E402
from paper_2006_05664_b200.evaluator import _op_args  # noqa: E402
from paper_2006_05664_b200.operators import parse_operator  # noqa: E402
from paper_2006_05664_b200.prebuild import family_instances  # noqa: E402


def main():
    spec = parse_operator(sys.argv[1])
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    inst = sorted(family_instances(spec))
    dev = capi.Device(0)
    op = dev.prepare(**_op_args(spec))
    t0 = time.perf_counter()
    res, bad = [], []
    for _fam, _batched, kn in inst:
        t = dev.trial(op, kn, warmup=3, reps=reps)
        if t.ok:
            res.append((t.tflops, kn))
        elif t.status != capi.INVALID_CONFIG:
            bad.append((kn, t.status, t.message[:80]))
    res.sort(reverse=True)
    print(f"{spec.id()}: {len(inst)} instances, {len(res)} timed, {len(bad)} failed, "
          f"{time.perf_counter() - t0:.0f} s")
    # re-time the leaders longer (noise must not decide the ranking)
    final = []
    for _, kn in res[:top]:
        k = dev.kernel(op, kn)
        ms = min(k.time(warmup=3, reps=100) for _ in range(3))
        k.close()
        final.append((spec.flops() / ms / 1e9, kn))
    final.sort(reverse=True)
    for tf, kn in final:
        print(f"  {tf:8.1f} TFLOP/s  {','.join(map(str, kn))}")
    for b in bad[:10]:
        print("  FAILED", b)


if __name__ == "__main__":
    main()
