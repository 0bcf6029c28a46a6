"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import csv, sys
from collections import defaultdict
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0].isdigit()]
agg = defaultdict(lambda: [0, 0.0])
for r in rows:
    agg[r[4][:60]][0] += 1
    agg[r[4][:60]][1] += float(r[-1])
tot = sum(v[1] for v in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:60s} {n:5d} {t / 1e6:10.2f} ms  {100 * t / tot:5.1f}%")
