"""Top SASS instructions by warp-stall samples from an ncu source page
(ncu -i X.ncu-rep --page source --csv --print-source sass > X.csv).
Usage: python tools/sass_hot.py X.csv [top]"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    hdr = rows[1]
    data = rows[2:]
    ia, isrc, isamp = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(float(r[isamp] or 0) for r in data)
    print(f"total samples {tot:.0f}")
    by = sorted(data, key=lambda r: -float(r[isamp] or 0))
    for r in by[:top]:
        s = float(r[isamp] or 0)
        reasons = sorted(((float(r[i] or 0), hdr[i][6:]) for i in stall_cols), reverse=True)[:3]
        rs = " ".join(f"{n}:{v:.0f}" for v, n in reasons if v > 0)
        print(f"{r[ia]:>6s} {100 * s / tot:5.1f}%  {r[isrc][:70]:70s} {rs}")


if __name__ == "__main__":
    main()
