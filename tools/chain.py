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

import paper_2107_09801_b200 as P  # noqa: E402
from paper_2107_09801_b200.chain import run_chain  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=14)
    ap.add_argument("--rounds", type=int, default=4)
    ap.add_argument("--seconds", type=float, default=30.0)
    ap.add_argument("--walks", type=int, default=0)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--devices", type=int, nargs="+", default=[0])
    args = ap.parse_args()
    import torch
    nsm = torch.cuda.get_device_properties(args.devices[0]).multi_processor_count
    walks = args.walks or nsm * len(args.devices)     # one wave of walk CTAs per GPU
    L = (1 << args.m) - 1
    p = P.default_params(L)
    p.seed = args.seed
    p.stop = P.StopCondition(max_seconds=args.seconds)
    t0 = [time.perf_counter()]

    def report(r):
        print(json.dumps({"m": args.m, "round": r.round, "walks": walks, "devices": len(args.devices),
                          "seconds": args.seconds, "wall": time.perf_counter() - t0[0],
                          "round_best_psl": r.round_best_psl, "chain_best_psl": r.chain_best_psl,
                          "chain_best_mf": r.chain_best_mf, "nse": r.nse,
                          "switches": r.switches}), flush=True)
        t0[0] = time.perf_counter()

    run_chain(p, walks, args.rounds, devices=args.devices, on_round=report)


if __name__ == "__main__":
    main()
