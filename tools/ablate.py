"""Time ablated instances (debug builds) to split a kernel's launch time into
launch floor / prologue+epilogue / loads / MMA.  Each variant runs in its own
process (the variant is a compile flag read from the environment)."""
import os
import subprocess
import sys

CODE = r'''
import sys; sys.path.insert(0, ".")
from paper_2006_05664_b200 import capi
from paper_2006_05664_b200.evaluator import _op_args
from paper_2006_05664_b200.operators import parse_operator
spec = parse_operator(sys.argv[1]); kn = tuple(int(x) for x in sys.argv[2].split(","))
dev = capi.Device(0, "/tmp/opevo_ablate_cache"); op = dev.prepare(**_op_args(spec))
k = dev.kernel(op, kn)
print("%.3f" % (k.time(warmup=5, reps=100) * 1e3))
'''
NAMES = {0: "full kernel", 1: "exit at entry", 2: "no mainloop", 3: "no TMA (MMA only)", 4: "no MMA (TMA only)",
         6: "no C stores", 7: "no mainloop, no stores"}
for op, kn in [(a.split("@")[0], a.split("@")[1]) for a in sys.argv[1:]]:
    print(f"{op} knobs {kn}")
    for pdl in ("1", "0"):
        for ab in (0, 1, 2, 3, 4, 6, 7):
            env = dict(os.environ, OPEVO_EXTRA_FLAGS=f"-DOPEVO_ABLATE={ab}", OPEVO_NO_PDL="0" if pdl == "1" else "1")
            r = subprocess.run([sys.executable, "-c", CODE, op, kn], env=env, capture_output=True, text=True)
            val = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else ("ERR " + r.stderr.strip()[-120:])
            print(f"  pdl={pdl} {NAMES[ab]:22s} {val} us/launch")
