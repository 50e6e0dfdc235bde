"""Per-launch time of the same instances under the three timing modes
(0 graph, 2 gated stream, 1 cold L2), and cuBLAS (torch.matmul, stream loop
and CUDA graph) on the same shape for reference.
Usage: python tools/timing_modes.py matmul:1024,1024,1024 128,64,128,3,1,1 ..."""
import sys

sys.path.insert(0, ".")
from paper_2006_05664_b200 import capi  # noqa: E402
from paper_2006_05664_b200.evaluator import _op_args  # noqa: E402
from paper_2006_05664_b200.operators import parse_operator  # noqa: E402


def main():
    spec = parse_operator(sys.argv[1])
    dev = capi.Device(0)
    op = dev.prepare(**_op_args(spec))
    for a in sys.argv[2:]:
        kn = tuple(int(x) for x in a.split(","))
        k = dev.kernel(op, kn)
        res = []
        for mode in (0, 2, 0, 2, 1):
            us = k.time(warmup=3, reps=20, flush_l2=mode) * 1e3
            res.append(f"m{mode} {us:6.2f}us {spec.flops() / us / 1e6:6.1f}TF")
        print(kn, " | ".join(res))
        k.close()
    if spec.__class__.__name__ == "MatMulSpec":
        import torch
        a = torch.randn(spec.n, spec.k, device="cuda", dtype=torch.bfloat16)
        b = torch.randn(spec.m, spec.k, device="cuda", dtype=torch.bfloat16)
        for _ in range(10):
            torch.matmul(a, b.t())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(200):
            torch.matmul(a, b.t())
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 200
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            torch.matmul(a, b.t())
        torch.cuda.current_stream().wait_stream(s)
        with torch.cuda.graph(g):
            for _ in range(20):
                torch.matmul(a, b.t())
        g.replay()
        torch.cuda.synchronize()
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ug = e0.elapsed_time(e1) * 1e3 / 20
        print(f"cuBLAS stream loop {us:.2f}us {spec.flops() / us / 1e6:.1f}TF | graph {ug:.2f}us "
              f"{spec.flops() / ug / 1e6:.1f}TF")


if __name__ == "__main__":
    main()
