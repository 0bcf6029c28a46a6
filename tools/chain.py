#!/usr/bin/env python
"""Warm-start chains (the paper's repeated-restart protocol, README.md:90-91 /
PAPER.md:425-427): round r restarts every walk from the best sequence found
in round r-1 (search.hpp SearchParams.init), with fresh seeds, for T seconds.

  python tools/chain.py --m 14 --rounds 4 --seconds 30
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2107_09801_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=14)
    ap.add_argument("--rounds", type=int, default=4)
    ap.add_argument("--seconds", type=float, default=30.0)
    ap.add_argument("--walks", type=int, default=0)
    ap.add_argument("--seed", type=int, default=1)
    args = ap.parse_args()
    import torch
    walks = args.walks or torch.cuda.get_device_properties(0).multi_processor_count   # one wave
    ctx = P.Context(0)
    L = (1 << args.m) - 1
    best_seq, best_psl = None, None
    for r in range(args.rounds):
        p = P.default_params(L)
        p.seed = args.seed + r * walks
        p.stop = P.StopCondition(max_seconds=args.seconds)
        inits = None if best_seq is None else np.repeat(best_seq[None, :], walks, axis=0)
        t0 = time.perf_counter()
        recs = P.run_walks(p, walks, inits=inits, ctx=ctx, solutions=True)
        i = int(np.argmin([x.psl_best for x in recs]))
        if best_psl is None or recs[i].psl_best < best_psl:
            best_psl, best_seq = recs[i].psl_best, recs[i].solution_best.copy()
        rep = P.verify_sequence(best_seq, ctx)
        assert rep.psl == best_psl
        print(json.dumps({"m": args.m, "round": r + 1, "walks": walks, "seconds": args.seconds,
                          "wall": time.perf_counter() - t0, "round_best_psl": recs[i].psl_best,
                          "chain_best_psl": best_psl, "chain_best_mf": rep.merit_factor,
                          "nse": int(sum(x.nse for x in recs))}), flush=True)


if __name__ == "__main__":
    main()
