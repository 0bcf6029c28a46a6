"""How often would a certified (interval) scan need exact serial chains?

Walks a two-phase trajectory with the exact engine (scan_values on the device,
reference decision rules) and records, per step, the relative gap between the
best and second-best neighbour value and between value_step and value_local.
A step is "ambiguous" at tolerance eps when another neighbour (or value_local)
lies within eps * value_step of the argmin.

    python tools/gaps.py --length 262143 --steps 3000 --ls-lmt 300
"""
import argparse
import json
import sys
import os

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_09801_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--length", type=int, default=262143)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--ls-lmt", type=int, default=300)
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    L, n = a.length, a.n
    rng = np.random.default_rng(a.seed)
    seq = np.where(rng.integers(0, 2, L) == 1, 1, -1).astype(np.int8)
    table = P.build_table(seq).astype(np.int32)
    luts = {al: P.PowerTable(L, al).lut for al in (4, P.default_alpha2(L))}
    alpha = 4
    value_local = P.fitness(table, alpha)
    local = (seq.copy(), table.copy())
    unimproved = 0
    epss = [1e-12, 1e-10, 1e-9, 1e-8, 1e-6]
    stats = {ph: {"steps": 0, "gap12": [], "gaploc": [], "amb": {e: 0 for e in epss},
                  "amb_loc": {e: 0 for e in epss}} for ph in (1, 2)}
    phase = 1
    for step in range(a.steps):
        start = int(rng.integers(L))
        vals, _ = P.scan_values(seq, table, start, n, luts[alpha])
        v = vals[1:]
        i = int(np.argmin(v))
        v1 = v[i]
        v2 = np.partition(v, 1)[1]
        st = stats[phase]
        st["steps"] += 1
        st["gap12"].append(float((v2 - v1) / v1))
        st["gaploc"].append(float(abs(v1 - value_local) / value_local))
        for e in epss:
            st["amb"][e] += int(np.count_nonzero(v <= v1 * (1 + e)) > 1)
            st["amb_loc"][e] += int(abs(v1 - value_local) <= e * v1)
        P.apply_flip(seq, table, (start + 1 + i) % L)
        if v1 < value_local:
            value_local = v1
            local = (seq.copy(), table.copy())
            unimproved = 0
        elif v1 > value_local:
            unimproved += 1
            if unimproved > a.ls_lmt:
                seq, table = local[0].copy(), local[1].copy()
                for p in rng.choice(L, P.default_flip_lmt(L), replace=False):
                    P.apply_flip(seq, table, int(p))
                phase = 3 - phase
                alpha = 4 if phase == 1 else P.default_alpha2(L)
                value_local = P.fitness(table, alpha)
                local = (seq.copy(), table.copy())
                unimproved = 0
    out = {}
    for ph, st in stats.items():
        if not st["steps"]:
            continue
        g = np.array(st["gap12"])
        gl = np.array(st["gaploc"])
        out[ph] = {"steps": st["steps"],
                   "gap12_quantiles": {q: float(np.quantile(g, q)) for q in (0.001, 0.01, 0.1, 0.5)},
                   "gaploc_quantiles": {q: float(np.quantile(gl, q)) for q in (0.001, 0.01, 0.1, 0.5)},
                   "ambiguous_frac": {str(e): st["amb"][e] / st["steps"] for e in epss},
                   "ambiguous_local_frac": {str(e): st["amb_loc"][e] / st["steps"] for e in epss}}
    print(json.dumps({"L": L, "n": n, "ls_lmt": a.ls_lmt, "phases": out}, indent=1))


if __name__ == "__main__":
    main()
