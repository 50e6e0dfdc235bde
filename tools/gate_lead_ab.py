"""Early release of a batch's first device gate (OPEVO_GATE_LEAD): the
fitness a single-trial batch measures, and its wall time, with the gate
opened after the whole trial is queued (0) or after `lead` timed launches
(default 6).  Each setting runs in its own process (the library reads the
variable once), rounds alternate.
Usage: python tools/gate_lead_ab.py OP KNOBS [rounds]"""
import json
import os
import statistics
import subprocess
import sys

CODE = r'''
import json, sys, time, statistics
sys.path.insert(0, ".")
from paper_2006_05664_b200 import capi
from paper_2006_05664_b200.evaluator import _op_args
from paper_2006_05664_b200.operators import parse_operator
spec = parse_operator(sys.argv[1]); kn = tuple(int(x) for x in sys.argv[2].split(","))
dev = capi.Device(0); op = dev.prepare(**_op_args(spec))
fit, wall = [], []
for i in range(60):
    t0 = time.perf_counter()
    r = dev.trial_batch(op, [kn], warmup=3, reps=20, flush_l2=2)[0]
    wall.append(time.perf_counter() - t0)
    if i >= 10: fit.append(r.tflops)
print(json.dumps({"tflops": statistics.median(fit), "spread": [min(fit), max(fit)],
                  "wall_ms": 1e3 * statistics.median(wall[10:])}))
'''


def main():
    op, kn = sys.argv[1], sys.argv[2]
    rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    res = {0: [], 6: []}
    for _ in range(rounds):
        for lead in (0, 6):
            env = dict(os.environ, OPEVO_GATE_LEAD=str(lead))
            out = subprocess.run([sys.executable, "-c", CODE, op, kn], env=env, capture_output=True, text=True)
            res[lead].append(json.loads(out.stdout.strip().splitlines()[-1]))
    for lead, rs in res.items():
        print(f"{op} {kn} lead={lead}: fitness " + ", ".join(f"{r['tflops']:.1f} [{r['spread'][0]:.1f},{r['spread'][1]:.1f}]" for r in rs)
              + f"; single-trial batch wall {statistics.median(r['wall_ms'] for r in rs):.3f} ms")


if __name__ == "__main__":
    main()
