"""Stall samples of an ncu source page (--page source --csv --print-source cuda,sass)
attributed per SASS address (deduplicated over inline frames) to the innermost
function of psl_cert.cuh / psl_kernels.cu, with the stall-reason split.
usage: python tools/ncu_regions.py src.csv cert.cuh kernels.cu"""
import csv, re, sys
from collections import defaultdict

def funcs(path):
    """line -> enclosing function name (top-level definitions)."""
    names, cur = {}, "?"
    for i, l in enumerate(open(path), 1):
        if re.match(r"(?:template <[^>]*>\s*)?(?:__device__|__global__)", l):
            l2 = re.sub(r"__launch_bounds__\([^)]*\([^)]*\)[^)]*\)|__launch_bounds__\([^)]*\)", "", l)
            m = re.search(r"\b(\w+)\(", l2)
            if m:
                cur = m.group(1)
        names[i] = cur
    return names

src, certp, kernp = sys.argv[1:4]
fmap = {"psl_cert.cuh": funcs(certp), "psl_kernels.cu": funcs(kernp)}
rows = list(csv.reader(open(src)))
hdr = [r for r in rows if r and r[0] == "Line No"][0]
reasons = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "(Not Issued)" not in h]
seen = {}
f = cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0].isdigit():
        cur = (f, int(r[0]))
        continue
    if r[0] == "" and len(r) > 8 and r[2].startswith("0x"):
        addr = r[2]
        prio = 2 if cur[0] == "psl_cert.cuh" else (1 if cur[0] == "psl_kernels.cu" else 0)
        if addr not in seen or prio > seen[addr][0]:
            try:
                vals = [int(r[i] or 0) for i, _ in reasons]
                seen[addr] = (prio, cur, int(r[4] or 0), int(r[7] or 0), vals, r[3].strip())
            except ValueError:
                pass
agg = defaultdict(lambda: [0, 0, [0] * len(reasons)])
for prio, cur, s, n, vals, sass in seen.values():
    fn = fmap.get(cur[0], {}).get(cur[1], cur[0])
    key = f"{cur[0]}:{fn}"
    a = agg[key]
    a[0] += s; a[1] += n
    a[2] = [x + y for x, y in zip(a[2], vals)]
tot = sum(a[0] for a in agg.values()) or 1
for k, (s, n, vals) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:25]:
    top = sorted(zip(vals, [h[6:] for _, h in reasons]), reverse=True)[:4]
    print(f"{100*s/tot:5.1f}% inst {n:>12d}  {k:40s} " + " ".join(f"{h}:{100*v/max(s,1):.0f}%" for v, h in top))
