"""Summarise ncu reports (.ncu-rep) into profiles/ as JSON.
Usage: python tools/ncu_summary.py OUT.json NAME=report.ncu-rep[:flops[:algo_bytes]] ..."""
import csv
import io
import json
import re
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "l1tex__m_xbar2l1tex_read_bytes.sum", "sm__cycles_active.avg", "sm__cycles_elapsed.avg",
    "sm__cycles_elapsed.avg.per_second", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__cluster_dim_x",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3,
         "Ghz": 1, "Mhz": 1e-3}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                v = vals[i].replace(",", "")
                try:
                    x = float(v) * SCALE.get(units[i], 1)
                except ValueError:
                    x = v
                name = k
                if units[i] in ("byte", "Kbyte", "Mbyte", "Gbyte"):
                    name = k + "[bytes]"
                elif units[i] in ("ns", "us", "ms"):
                    name = k + "[us]"
                d[name] = x
        res.append(d)
    return res


def main():
    out = {}
    for arg in sys.argv[2:]:
        name, spec = arg.split("=", 1)
        parts = spec.split(":")
        rows = raw(parts[0])
        for r in rows:
            us = r.get("gpu__time_duration.sum[us]")
            if len(parts) > 1 and us:
                r["algorithmic_tflops_at_ncu_duration"] = float(parts[1]) / (us * 1e-6) / 1e12
            if len(parts) > 2:
                r["algorithmic_bytes"] = float(parts[2])
            r["dram_bytes"] = r.get("dram__bytes_read.sum[bytes]", 0) + r.get("dram__bytes_write.sum[bytes]", 0)
        out[name] = rows
    with open(sys.argv[1], "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1)[:3000])


if __name__ == "__main__":
    main()
