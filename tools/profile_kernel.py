"""Run one kernel instance a few times (target for ncu).
Usage: python tools/profile_kernel.py matmul:1024,1024,1024 128,64,128,3,1,1 [launches] [--tf32x3]"""
import sys

sys.path.insert(0, ".")
from paper_2006_05664_b200 import capi  # noqa: E402
from paper_2006_05664_b200.evaluator import _op_args  # noqa: E402
from paper_2006_05664_b200.operators import parse_operator  # noqa: E402


def main():
    x3 = "--tf32x3" in sys.argv
    argv = [a for a in sys.argv if a != "--tf32x3"]
    spec = parse_operator(argv[1])
    knobs = tuple(int(x) for x in argv[2].split(","))
    n = int(argv[3]) if len(argv) > 3 else 5
    dev = capi.Device(0)
    op = dev.prepare(dtype=capi.F32_TF32X3 if x3 else capi.BF16, **_op_args(spec))
    k = dev.kernel(op, knobs)
    print("rel err", k.check())
    for _ in range(n):
        k.run()
    ms = k.time(warmup=3, reps=50)
    print(f"{spec.id()} knobs={knobs}: {ms * 1e3:.2f} us/launch, {spec.flops() / ms / 1e9:.1f} TFLOP/s")


if __name__ == "__main__":
    main()
