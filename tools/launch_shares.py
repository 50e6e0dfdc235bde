"""Per-kernel launch counts and time shares from an ncu launch list
(ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv).
Cold, serialised launches: compare shares, not absolute times.
Usage: python tools/launch_shares.py launches.csv"""
import csv
import sys
from collections import defaultdict


def main():
    lines = [ln for ln in open(sys.argv[1]) if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    t = defaultdict(float)
    n = defaultdict(set)
    dram = defaultdict(float)
    for r in rows:
        k = r["Kernel Name"]
        n[k].add(r["ID"])
        v = float(r["Metric Value"].replace(",", "") or 0)
        if r["Metric Name"] == "gpu__time_duration.sum":
            t[k] += v * (1e-3 if r["Metric Unit"] == "ns" else 1.0)
        elif r["Metric Name"].startswith("dram__bytes"):
            dram[k] += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r["Metric Unit"], 1)
    tot = sum(t.values())
    for k in sorted(t, key=lambda x: -t[x]):
        print(f"{k:22s} launches={len(n[k]):5d} time_us={t[k]:10.1f} share={100 * t[k] / tot:5.1f}% "
              f"dram_MB={dram[k] / 1e6:9.1f}")


if __name__ == "__main__":
    main()
