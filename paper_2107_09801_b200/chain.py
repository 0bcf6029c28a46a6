"""Warm-start chains: the paper's repeated-restart quality protocol.

The reference runs it as a shell loop around its CLI (proj/README.md:90-91:
`pslopt solve --init best.txt ...` again and again), and the paper restarts
its best runs 4x from their own best sequences.  Round r
here runs `walks` independent walks (seeds seed0 + r * walks + w) for the same
stop condition; from round 2 on every walk starts from the best sequence found
so far (SearchParams.init, search.hpp:41).  Walks are spread over `devices`
(psl_run_walks_multi: one host thread and context per GPU, records gathered on
the host); the chain's best only ever improves (the minimum over rounds, ties
keep the earlier sequence).
"""
from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Optional, Sequence

import numpy as np

from . import pslopt as P


@dataclass
class ChainRound:
    round: int
    seeds: list
    round_best_psl: int
    round_best_walk: int
    chain_best_psl: int
    chain_best_mf: float
    nse: int
    switches: int
    records: list


def run_chain(params: P.SearchParams, walks: int, rounds: int,
              devices: Sequence[int] = (0,), init: Optional[np.ndarray] = None,
              on_round=None) -> tuple[list[ChainRound], np.ndarray]:
    """Runs `rounds` rounds of `walks` walks; returns (per-round summaries, the
    chain's best sequence).  `init` seeds round 1 (else random starts);
    `on_round(ChainRound)` is called after each round."""
    p0 = P.validate_params(params)
    L = p0.length
    best_seq = None if init is None else np.ascontiguousarray(init, np.int8).copy()
    best_psl = None
    out = []
    for r in range(rounds):
        seeds = [p0.seed + r * walks + w for w in range(walks)]
        p = replace(p0, init=None)
        inits = None if best_seq is None else best_seq      # one (L,) start for every walk
        if len(devices) > 1:
            recs, bw, _ = P.run_walks_multi(p, walks, devices=list(devices), seeds=seeds,
                                            inits=inits)
        else:
            ctx = P.default_context() if devices[0] == 0 else P.Context(devices[0])
            recs = P.run_walks(p, walks, seeds=seeds, inits=inits, ctx=ctx)
            bw = min(range(walks), key=lambda i: (recs[i].psl_best, i))
        if best_psl is None or recs[bw].psl_best < best_psl:
            best_psl, best_seq = recs[bw].psl_best, recs[bw].solution_best.copy()
        t = P.build_table(best_seq)
        assert P.psl(t) == best_psl, "chain best does not re-verify"
        cr = ChainRound(r + 1, seeds, int(recs[bw].psl_best), int(bw), int(best_psl),
                        float(P.merit_factor(t)), int(sum(x.nse for x in recs)),
                        int(sum(x.switches for x in recs)), recs)
        out.append(cr)
        if on_round:
            on_round(cr)
    assert best_seq is not None and len(best_seq) == L
    return out, best_seq
