"""Print selected raw metrics of an ncu report.
Usage: python tools/ncu_metrics.py X.ncu-rep [regex]"""
import csv
import io
import re
import subprocess
import sys

DEFAULT = (r"(gpu__time_duration.sum|dram__bytes_read.sum$|dram__bytes_write.sum$|lts__t_sector_hit_rate.pct"
           r"|l1tex__m_xbar2l1tex_read_bytes.sum$|sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
           r"|lts__throughput.avg.pct|launch__grid_size|sm__cycles_active.avg$|launch__shared_mem_per_block_dynamic"
           r"|launch__cluster_dim_x|l1tex__m_l1tex2xbar_write_bytes.sum$)")


def main():
    rep = sys.argv[1]
    pat = re.compile(sys.argv[2] if len(sys.argv) > 2 else DEFAULT)
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        for i, h in enumerate(hdr):
            if pat.search(h):
                print(f"{h:75s} {vals[i]} {units[i]}")


if __name__ == "__main__":
    main()
