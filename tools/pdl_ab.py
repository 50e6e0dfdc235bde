"""A/B of programmatic dependent launch on a few instances (separate processes
because the PDL switch is read at launch time)."""
import os
import subprocess
import sys

CASES = [("matmul:1024,1024,1024", "128,64,256,2,1,1"), ("matmul:1024,1024,1024", "128,64,128,3,1,1"),
         ("matmul:1024,1024,1024", "128,128,128,3,1,1"), ("matmul:1024,1024,1024", "256,64,128,3,1,1"),
         ("matmul:4096,4096,4096", "256,256,64,3,1,1"), ("batchmatmul:960,128,64,128", "128,64,64,2,1,1")]
for op, kn in CASES:
    for pdl in ("0", "1"):
        env = dict(os.environ, OPEVO_NO_PDL="0" if pdl == "1" else "1")
        out = subprocess.run([sys.executable, "tools/profile_kernel.py", op, kn, "1"], env=env,
                             capture_output=True, text=True).stdout.strip().splitlines()
        print(f"pdl={pdl}", out[-1] if out else "FAILED")
