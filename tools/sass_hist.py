"""Summarise an ncu source page (SASS) by opcode and by hot address ranges.
usage: ncu -i rep --page source --csv --print-source sass | python tools/sass_hist.py"""
import csv, sys, collections
rows = list(csv.reader(sys.stdin))
hdr = None
data = []
for r in rows:
    if len(r) > 3 and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
ops = collections.Counter()
stall = collections.Counter()
tot = 0
for d in data:
    n = int(d.get("Instructions Executed", "0") or 0)
    src = d["Source"].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    ops[op] += n
    tot += n
    stall[op] += int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
print(f"total warp instructions: {tot:.4g}")
for op, n in ops.most_common(25):
    print(f"{op:10s} {n:14d} {100.0*n/tot:6.2f}%  stall-samples {stall[op]}")
