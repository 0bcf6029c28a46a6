"""Group an ncu SASS source page into straight-line regions (same execution
count) and print the heaviest ones with their opcode mix."""
import csv, sys, collections
rows = list(csv.reader(sys.stdin))
hdr = None
out = []
for r in rows:
    if len(r) > 3 and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        out.append((d["Source"].strip(), int(d["Instructions Executed"] or 0)))
regions = []
cur = None
for s, n in out:
    if n == 0:
        continue
    if cur and cur[0] == n:
        cur[1].append(s)
    else:
        cur = [n, [s]]
        regions.append(cur)
tot = sum(n * len(i) for n, i in regions)
show = int(sys.argv[1]) if len(sys.argv) > 1 else 8
dump = int(sys.argv[2]) if len(sys.argv) > 2 else -1
for idx, (n, ins) in enumerate(sorted(regions, key=lambda r: -r[0] * len(r[1]))[:show]):
    ops = collections.Counter((i.split()[1] if i.startswith("@") else i.split()[0]).split(".")[0] for i in ins)
    print(f"[{idx}] count={n:>10d} len={len(ins):4d} share={100*n*len(ins)/tot:5.1f}%  {dict(ops.most_common(9))}")
    if idx == dump:
        print("\n".join(ins))
