#!/usr/bin/env python
"""Best PSL at fixed wall time (BASELINE.json metric part 2, configs 4-5).

For each m, runs W independent walks (seed0 + w, one CTA each) of
the two-phase search for T seconds on one B200 (max_seconds stop, device
clock), and optionally the single-exponent ablations (alpha1 = alpha2 = 4 and
alpha1 = alpha2 = default alpha2, reference main.cpp:145-151).  Prints one JSON
line per (m, mode): best / mean PSL, PSL / sqrt(L), NSE.

  python tools/quality.py --m 14 16 18 20 --seconds 30 [--ablation]
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2107_09801_b200 as P  # noqa: E402

PAPER_BEST = {14: 101, 15: 146, 16: 209, 17: 301, 18: 434, 19: 628, 20: 901}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, nargs="+", default=[14, 16, 18, 20])
    ap.add_argument("--seconds", type=float, default=30.0)
    ap.add_argument("--walks", type=int, default=0)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--ablation", action="store_true")
    ap.add_argument("--modes", nargs="+", default=None,
                    help="subset of two-phase single-alpha1 single-alpha2")
    ap.add_argument("--devices", type=int, nargs="+", default=[0],
                    help="GPUs of this node (walks split over them, psl_run_walks_multi)")
    args = ap.parse_args()
    ctx = P.Context(args.devices[0])
    import torch
    nsm = torch.cuda.get_device_properties(args.devices[0]).multi_processor_count
    # one walk CTA per SM (the certified kernel) on every GPU
    walks = args.walks or nsm * len(args.devices)
    for m in args.m:
        L = (1 << m) - 1
        a2 = P.default_alpha2(L)
        modes = [("two-phase", 4, a2)]
        if args.ablation:
            modes += [("single-alpha1", 4, 4), ("single-alpha2", a2, a2)]
        if args.modes:
            modes = [x for x in [("two-phase", 4, a2), ("single-alpha1", 4, 4),
                                 ("single-alpha2", a2, a2)] if x[0] in args.modes]
        for name, a1, b2 in modes:
            p = P.SearchParams(length=L, seed=args.seed, alpha1=a1, alpha2=b2, ls_lmt=2000,
                               flip_lmt=10, n_lmt=min(L, 1024),
                               stop=P.StopCondition(max_seconds=args.seconds))
            t0 = time.perf_counter()
            seeds = [args.seed + w for w in range(walks)]
            if len(args.devices) > 1:
                recs, _, _ = P.run_walks_multi(p, walks, devices=args.devices, seeds=seeds)
            else:
                recs = P.run_walks(p, walks, seeds=seeds, ctx=ctx, solutions=True)
            wall = time.perf_counter() - t0
            psls = np.array([r.psl_best for r in recs])
            best = int(np.argmin(psls))
            # re-verify the winner from a fresh table build
            t = P.build_table(recs[best].solution_best, ctx)
            assert P.psl(t) == recs[best].psl_best
            line = {"m": m, "L": L, "mode": name, "alpha1": a1, "alpha2": b2, "walks": walks,
                    "seconds": args.seconds, "wall_seconds": wall,
                    "best_psl": int(psls.min()), "mean_psl": float(psls.mean()),
                    "best_psl_over_sqrtL": float(psls.min() / math.sqrt(L)),
                    "mean_psl_over_sqrtL": float(psls.mean() / math.sqrt(L)),
                    "nse_total": int(sum(r.nse for r in recs)),
                    "devices": len(args.devices),
                    "walks_switched": int(sum(1 for r in recs if r.switches > 0)),
                    "switches_total": int(sum(r.switches for r in recs)),
                    "steps_mean": float(np.mean([r.steps for r in recs])),
                    "best_walk_seed": int(recs[best].seed), "best_mf": recs[best].merit_factor,
                    "paper_best_4day_a100": PAPER_BEST.get(m)}
            print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
