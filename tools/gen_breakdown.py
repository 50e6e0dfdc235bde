"""Where one OpEvo generation's wall time goes on the GPU evaluator (no
profiler overhead): L2 flush, ask, mapping + staging, the C trial batch
(bind, check phase, sync, timed phase, sync), tell + record.
Usage: python tools/gen_breakdown.py [op] [generations]"""
import statistics
import sys
import time

sys.path.insert(0, ".")


def main():
    op_id = sys.argv[1] if len(sys.argv) > 1 else "matmul:1024,1024,1024"
    gens = int(sys.argv[2]) if len(sys.argv) > 2 else 60
    from paper_2006_05664_b200 import EngineConfig, OpEvo, parse_operator
    from paper_2006_05664_b200.evaluator import EvalSettings, GpuEvaluator
    from paper_2006_05664_b200.logs import TrialRecorder
    from paper_2006_05664_b200.mapping import gpu_operator_space

    spec = parse_operator(op_id)
    space = gpu_operator_space(spec)
    ev = GpuEvaluator(spec, space, 0, EvalSettings(preload_family=True))
    eng = OpEvo(space, EngineConfig(seed=0, budget=8 * (gens + 5)))
    rec = TrialRecorder(space)
    acc = {}

    def timed(name, fn):
        def w(*a, **k):
            t = time.perf_counter()
            try:
                return fn(*a, **k)
            finally:
                acc.setdefault(name, []).append(time.perf_counter() - t)
        return w

    ev.dev.trial_batch = timed("trial_batch (C)", ev.dev.trial_batch)
    ev.precompile = timed("precompile", ev.precompile)
    rows = []
    for g in range(gens + 5):
        acc.clear()
        t = [time.perf_counter()]
        ev.dev.flush_l2()
        t.append(time.perf_counter())
        a = eng.ask()
        t.append(time.perf_counter())
        fits = ev.evaluate(a.configs)
        t.append(time.perf_counter())
        eng.tell(list(zip(a.configs, fits)))
        for c, f, e in zip(a.configs, fits, ev.last_extras):
            rec.record(c, f, e)
        t.append(time.perf_counter())
        if g >= 5:
            tb = sum(acc.get("trial_batch (C)", [0]))
            pc = sum(acc.get("precompile", [0]))
            rows.append({"flush": t[1] - t[0], "ask": t[2] - t[1], "evaluate": t[3] - t[2],
                         "  trial_batch (C)": tb, "  precompile": pc,
                         "  rest of evaluate (map, python)": t[3] - t[2] - tb - pc,
                         "tell+record": t[4] - t[3], "total": t[4] - t[0]})
    print(f"{op_id}: {gens} generations (median / mean ms)")
    for k in rows[0]:
        v = [r[k] * 1e3 for r in rows]
        print(f"  {k:34s} {statistics.median(v):7.3f} {statistics.mean(v):7.3f}")
    ev.close()


if __name__ == "__main__":
    main()
