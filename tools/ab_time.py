"""A/B device timing of libpslb200 variants, one process per measurement,
alternating between the variants (the GPU's clock state is shared).

usage: python tools/ab_time.py libA.so libB.so [rounds] [-- step_time.py args]
       (default step_time args: --walks 444 --steps 10 --mode auto)"""
import json
import os
import subprocess
import sys

argv = sys.argv[1:]
extra = ["--walks", "444", "--steps", "10", "--mode", "auto"]
if "--" in argv:
    i = argv.index("--")
    argv, extra = argv[:i], argv[i + 1:]
libs = argv[:2]
rounds = int(argv[2]) if len(argv) > 2 else 3
here = os.path.dirname(os.path.abspath(__file__))
res = {lib: [] for lib in libs}
for r in range(rounds):
    for lib in libs:
        p = subprocess.run([sys.executable, os.path.join(here, "step_time.py")] + extra,
                           env={**os.environ, "PSLB200_LIB": lib}, capture_output=True, text=True)
        lines = p.stdout.strip().splitlines()
        if p.returncode or not lines:
            print(f"{lib}: failed: {p.stderr[-800:]}")
            continue
        d = json.loads(lines[-1])
        res[lib].append(round(d["auto_ms_per_step"], 3))
for lib in libs:
    v = sorted(res[lib])
    if v:
        print(f"{os.path.basename(lib)} {' '.join(extra)}: median {v[len(v) // 2]:.3f} ms/step  all {res[lib]}")
