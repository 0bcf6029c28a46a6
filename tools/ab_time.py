"""A/B device timing of libpslb200 variants in one process each, alternating.
usage: python tools/ab_time.py libA.so libB.so [rounds] [steps]"""
import json, os, subprocess, sys
libs = sys.argv[1:3]
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
steps = sys.argv[4] if len(sys.argv) > 4 else "5"
res = {l: [] for l in libs}
for r in range(rounds):
    for l in libs:
        out = subprocess.run([sys.executable, "tools/step_time.py", "--walks", "148", "--steps", steps,
                              "--mode", "auto"], env={**os.environ, "PSLB200_LIB": l},
                             capture_output=True, text=True).stdout.strip().splitlines()[-1]
        res[l].append(round(json.loads(out)["auto_ms_per_step"], 3))
for l in libs:
    v = sorted(res[l])
    print(f"{l}: median {v[len(v)//2]:.3f} ms/step  all {res[l]}")
