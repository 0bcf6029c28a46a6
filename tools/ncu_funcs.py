"""Instructions and stall samples of an ncu source page grouped by the enclosing
device function (psl_cert.cuh / psl_kernels.cu helpers; the kernel body itself as
'run_kernel').  usage: python tools/ncu_funcs.py report.ncu-rep"""
import csv, io, re, subprocess, sys, collections, os
rep = sys.argv[1]
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
def func_map(path):
    lines = open(path).read().splitlines()
    cur, out = "(top)", {}
    for i, l in enumerate(lines, 1):
        m = re.match(r"^(?:template <[^>]*>\s*)?(?:__device__|__global__)[^(]*?(\w+)\(", l)
        if m:
            cur = m.group(1)
        out[i] = cur
    return out
maps = {f: func_map(os.path.join(HERE, "paper_2107_09801_b200", "csrc", f))
        for f in ("psl_cert.cuh", "psl_kernels.cu")}
agg = collections.defaultdict(lambda: [0, 0])
file = None
hdr = None
for r in csv.reader(io.StringIO(src)):
    if not r:
        continue
    if r[0] == "File Path":
        file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0].isdigit() and len(r) == len(hdr):
        d = dict(zip(hdr[4:], r[4:]))
        try:
            n, s = int(d.get("Instructions Executed") or 0), int(d.get("Warp Stall Sampling (All Samples)") or 0)
        except ValueError:
            continue
        fn = maps.get(file, {}).get(int(r[0]), file)
        agg[fn][0] += n
        agg[fn][1] += s
tn = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"{'function':28s} {'instr %':>8s} {'stall samples %':>16s}")
for k, (n, s) in sorted(agg.items(), key=lambda x: -x[1][1])[:22]:
    print(f"{k:28s} {100*n/tn:8.1f} {100*s/ts:16.1f}")
