"""Per-CUDA-source-line stall samples / executed warp instructions of an ncu report.
usage: ncu -i rep --page source --csv --print-source cuda,sass | python tools/ncu_lines.py [N]"""
import csv, sys
rows = csv.reader(sys.stdin)
file = None
out = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        file = r[1].split("/")[-1]
        continue
    if r[0].isdigit() and len(r) > 7:
        try:
            s, n = int(r[4]), int(r[7])
        except ValueError:
            continue
        out.append((s, n, file, int(r[0]), r[1].strip()[:80]))
tot = sum(o[0] for o in out) or 1
N = int(sys.argv[1]) if len(sys.argv) > 1 else 40
for s, n, f, ln, src in sorted(out, reverse=True)[:N]:
    print(f"{100*s/tot:5.1f}% {n:>12d} {f}:{ln:<5d} {src}")
