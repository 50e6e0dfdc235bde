"""Quick sweep of kernel knobs on one shape; prints TFLOP/s per instance and
torch.matmul (cuBLAS) for comparison.  Usage: python tools/gpu_probe.py"""
import json
import sys
import time

sys.path.insert(0, ".")
from paper_2006_05664_b200 import capi  # noqa: E402


def main():
    shape = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1024,1024,1024").split(","))
    rows, cols, depth = shape
    dev = capi.Device(0)
    op = dev.prepare(capi.MATMUL, rows=rows, cols=cols, depth=depth)
    out = []
    for bm in (128, 256):
        for bn in (64, 128, 256):
            for bk in (64, 128):
                for st in (2, 3, 4, 6):
                    for split in (1, 2, 4):
                        for cl in (1, 2, 4):
                            kn = (bm, bn, bk, st, split, cl)
                            t = dev.trial(op, kn, warmup=3, reps=50)
                            if t.status == capi.INVALID_CONFIG:
                                continue
                            out.append((t.tflops, kn, t.status, t.rel_err, t.message[:80]))
    out.sort(reverse=True)
    for r in out[:25]:
        print("%.1f TFLOP/s  knobs=%s status=%d rel=%.2e %s" % r)
    bad = [r for r in out if r[2] != 0]
    print("non-ok:", len(bad), bad[:5])
    import torch
    a = torch.randn(rows, depth, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(cols, depth, device="cuda", dtype=torch.bfloat16)
    for _ in range(10):
        torch.matmul(a, b.t())
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(50):
            torch.matmul(a, b.t())
    g.replay()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    print("cuBLAS torch.matmul: %.1f TFLOP/s (%.2f us)" % (2 * rows * cols * depth / ms / 1e9, ms * 1e3))


if __name__ == "__main__":
    main()
