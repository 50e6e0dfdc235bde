"""cProfile of the bench generation loop (host overhead per generation).
Usage: python tools/profile_bench.py [op] [generations]"""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")


def main():
    op_id = sys.argv[1] if len(sys.argv) > 1 else "matmul:1024,1024,1024"
    gens = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    from paper_2006_05664_b200 import EngineConfig, OpEvo, parse_operator
    from paper_2006_05664_b200.evaluator import GpuEvaluator
    from paper_2006_05664_b200.logs import TrialRecorder
    from paper_2006_05664_b200.mapping import gpu_operator_space

    spec = parse_operator(op_id)
    space = gpu_operator_space(spec)
    ev = GpuEvaluator(spec, space, 0)
    eng = OpEvo(space, EngineConfig(seed=0, budget=8 * (gens + 5)))
    rec = TrialRecorder(space)

    def gen():
        ev.dev.flush_l2()
        a = eng.ask()
        fits = ev.evaluate(a.configs)
        eng.tell(list(zip(a.configs, fits)))
        for c, f, e in zip(a.configs, fits, ev.last_extras):
            rec.record(c, f, e)

    for _ in range(5):
        gen()
    t0 = time.perf_counter()
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(gens):
        gen()
    pr.disable()
    dt = time.perf_counter() - t0
    print(f"{gens} generations: {1e3 * dt / gens:.3f} ms/generation (under cProfile)")
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)
    ev.close()


if __name__ == "__main__":
    main()
