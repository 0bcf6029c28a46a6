"""A/B check of the certified scan against the exact sweep: same walks, both
scan modes, records + best sequences must be identical; prints wall time and
the certified/refined/chain step counts.

    python tools/cert_check.py --length 1048575 --walks 296 --steps 10
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_09801_b200 as P  # noqa: E402


def run(ctx, mode, params, walks):
    ctx.set_scan_mode(mode)
    before = ctx.scan_stats()
    t0 = time.perf_counter()
    recs = P.run_walks(params, n_walks=walks, ctx=ctx)
    dt = time.perf_counter() - t0
    after = ctx.scan_stats()
    return recs, dt, {k: after[k] - before[k] for k in after}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--length", type=int, default=65535)
    ap.add_argument("--walks", type=int, default=8)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--ls-lmt", type=int, default=None)
    ap.add_argument("--alpha2", type=int, default=None)
    ap.add_argument("--n-lmt", type=int, default=None)
    ap.add_argument("--auto-only", action="store_true")
    a = ap.parse_args()
    ctx = P.Context(0)
    p = P.default_params(a.length)
    p.seed = a.seed
    if a.ls_lmt is not None:
        p.ls_lmt = a.ls_lmt
    if a.alpha2 is not None:
        p.alpha2 = a.alpha2
    if a.n_lmt is not None:
        p.n_lmt = a.n_lmt
    p.stop = P.StopCondition(max_nse=1 + a.steps * p.n_lmt)
    out = {"L": a.length, "walks": a.walks, "steps": a.steps, "n_lmt": p.n_lmt}
    ra, ta, sa = run(ctx, ctx.SCAN_AUTO, p, a.walks)
    out["auto_s"] = ta
    out["auto_stats"] = sa
    out["auto_nse_per_s"] = sum(r.nse for r in ra) / ta
    if not a.auto_only:
        re_, te, se = run(ctx, ctx.SCAN_EXACT, p, a.walks)
        out["exact_s"] = te
        out["exact_stats"] = se
        out["exact_nse_per_s"] = sum(r.nse for r in re_) / te
        same = True
        for x, y in zip(ra, re_):
            fx = (x.nse, x.psl_best, x.energy, x.steps, x.switches, x.status)
            fy = (y.nse, y.psl_best, y.energy, y.steps, y.switches, y.status)
            if fx != fy or not np.array_equal(x.solution_best, y.solution_best):
                same = False
                out.setdefault("mismatch", []).append({"seed": x.seed, "auto": fx, "exact": fy})
        out["identical"] = same
        out["speedup"] = te / ta
    print(json.dumps(out))


if __name__ == "__main__":
    main()
