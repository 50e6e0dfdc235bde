"""ncu --set full capture of a list of kernel instances -> per-launch DRAM /
L2->SM traffic and tensor-pipe activity, merged into profiles/ncu_summary.json
(the `roofline.traffic` source of bench.py, keyed "operator|knobs").

Run on the GPU box (one GPU; ncu replays every kernel ~40 times):
    python tools/ncu_instances.py profiles/round2/ncu_instances.txt gpurun_out/ncu_update.json
then here:
    python tools/ncu_instances.py --merge gpurun_out/ncu_update.json

Each line of the list: ``operator|knobs`` (e.g. ``matmul:1024,1024,1024|128,64,128,3,...``),
the operator prefixed ``tf32x3:`` for the 3xTF32 family; ``#`` starts a comment.
"""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(REPO, "tools"))
from ncu_summary import raw  # noqa: E402

NCU = "/usr/local/cuda/bin/ncu"
SUMMARY = os.path.join(REPO, "profiles", "ncu_summary.json")


def capture(key: str, outdir: str) -> dict:
    op, knobs = key.split("|")
    x3 = op.startswith("tf32x3:")
    opname = op[len("tf32x3:"):] if x3 else op
    tag = (op + "_" + knobs).replace(":", "_").replace(",", "-")
    rep = os.path.join(outdir, "ncu_" + tag)
    cmd = [NCU, "--set", "full", "--clock-control", "none", "-k", "regex:opevo_gemm", "-s", "3",
           "-c", "1", "-f", "-o", rep, sys.executable, os.path.join(REPO, "tools", "profile_kernel.py"),
           opname, knobs, "3"] + (["--tf32x3"] if x3 else [])
    env = dict(os.environ, OPEVO_LINEINFO="1")
    done = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600)
    if done.returncode != 0 or not os.path.exists(rep + ".ncu-rep"):
        return {"error": (done.stdout + done.stderr)[-800:]}
    r = raw(rep + ".ncu-rep")[0]
    if os.environ.get("KEEP_NCU_REP") != "1":
        os.remove(rep + ".ncu-rep")       # reports are MBs each; the summary is what travels back
    return {"name": tag,
            "dram_bytes": r.get("dram__bytes_read.sum[bytes]", 0) + r.get("dram__bytes_write.sum[bytes]", 0),
            "ncu_us": r.get("gpu__time_duration.sum[us]"),
            "l2_to_sm_bytes": r.get("l1tex__m_xbar2l1tex_read_bytes.sum[bytes]"),
            "tensor_active_pct": r.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
            "grid": r.get("launch__grid_size"), "cluster_x": r.get("launch__cluster_dim_x"),
            "smem_dynamic": r.get("launch__shared_mem_per_block_dynamic[bytes]"),
            "report": os.path.basename(rep) + ".ncu-rep"}


def merge(update_path: str) -> None:
    with open(SUMMARY) as fh:
        summ = json.load(fh)
    with open(update_path) as fh:
        upd = json.load(fh)
    n = 0
    for key, v in upd.items():
        if "error" in v:
            print("skip", key, v["error"][-200:])
            continue
        summ["kernels"][key] = v
        n += 1
    with open(SUMMARY, "w") as fh:
        json.dump(summ, fh, indent=1)
    print(f"merged {n} instances into {SUMMARY}")


def main():
    if sys.argv[1] == "--merge":
        merge(sys.argv[2])
        return
    keys = []
    with open(sys.argv[1]) as fh:
        for ln in fh:
            ln = ln.split("#", 1)[0].strip()
            if ln:
                keys.append(ln)
    out_path = sys.argv[2]
    outdir = os.path.dirname(out_path) or "."
    res = {}
    for key in keys:
        res[key] = capture(key, outdir)
        print(key, {k: res[key].get(k) for k in ("dram_bytes", "ncu_us", "tensor_active_pct")}, flush=True)
        with open(out_path, "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
