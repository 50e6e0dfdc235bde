"""Summarise OPEVO_PROFILE_BATCH=1 lines (stderr of any run) per batch size:
median ms of each C-side phase of opevo_trial_batch.
Usage: python tools/batch_phases.py LOG"""
import collections
import re
import statistics
import sys

rows = collections.defaultdict(lambda: collections.defaultdict(list))
pat = re.compile(r"\[batch (\d+)\] (.*) ms")
for line in open(sys.argv[1]):
    m = pat.search(line)
    if not m:
        continue
    parts = m.group(2).split()
    for name, val in zip(parts[::2], parts[1::2]):
        rows[int(m.group(1))][name].append(float(val))
for n in sorted(rows):
    r = rows[n]
    cnt = len(next(iter(r.values())))
    tot = sum(statistics.median(v) for v in r.values())
    print(f"batch {n} ({cnt} batches): " + "  ".join(f"{k} {statistics.median(v):.3f}" for k, v in r.items())
          + f"  | sum of medians {tot:.3f} ms")
