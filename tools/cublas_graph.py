"""cuBLAS / cuDNN reference point: torch.matmul / bmm / conv2d (channels-last)
of an operator's shape, bf16, R back-to-back launches captured in one CUDA
graph (the same timing the roofline re-time of bench.py uses).
Usage: python tools/cublas_graph.py OP [R]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2006_05664_b200.operators import BatchMatMulSpec, Conv2dSpec, parse_operator  # noqa: E402


def main():
    spec = parse_operator(sys.argv[1])
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
    dev = torch.device("cuda", 0)
    if isinstance(spec, Conv2dSpec):
        x = torch.randn(spec.batch, spec.in_channels, spec.in_height, spec.in_width, device=dev,
                        dtype=torch.bfloat16).to(memory_format=torch.channels_last)
        w = torch.randn(spec.out_channels, spec.in_channels, spec.kernel_h, spec.kernel_w, device=dev,
                        dtype=torch.bfloat16).to(memory_format=torch.channels_last)
        fn = lambda: torch.nn.functional.conv2d(x, w, stride=spec.stride, padding=spec.padding)  # noqa: E731
    elif isinstance(spec, BatchMatMulSpec):
        a = torch.randn(spec.b, spec.n, spec.k, device=dev, dtype=torch.bfloat16)
        b = torch.randn(spec.b, spec.m, spec.k, device=dev, dtype=torch.bfloat16)
        fn = lambda: torch.bmm(a, b.transpose(1, 2))  # noqa: E731
    else:
        a = torch.randn(spec.n, spec.k, device=dev, dtype=torch.bfloat16)
        b = torch.randn(spec.m, spec.k, device=dev, dtype=torch.bfloat16)
        fn = lambda: torch.matmul(a, b.t())  # noqa: E731
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            fn()
    res = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g.replay()
        torch.cuda.synchronize()
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        res.append(spec.flops() / ms / 1e9)
    res.sort()
    print(f"cuBLAS {spec.id()}: median {res[2]:.1f} TFLOP/s (min {res[0]:.1f} max {res[-1]:.1f}), "
          f"{reps} launches per graph")


if __name__ == "__main__":
    main()
