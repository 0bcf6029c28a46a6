"""Warm-start chains (paper_2107_09801_b200/chain.py; the paper's repeated
restart protocol, run by the reference as a shell loop over
`pslopt solve --init`, proj/README.md:90-91).  Round r + 1 starts every walk
from the best sequence of rounds 1..r: each round's walk records must equal
the CPU oracle's run_search with that init (pinned to the reference), the
chain's best PSL never increases, and splitting the walks over two device
contexts changes nothing."""
import numpy as np
import pytest

from oracle import oracle_py as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("L,walks,rounds,max_nse", [(257, 4, 3, 20000), (4095, 3, 3, 30000)])
def test_chain_rounds_match_oracle(engine, L, walks, rounds, max_nse):
    from paper_2107_09801_b200.chain import run_chain
    a2 = engine.default_alpha2(L)
    n = min(L, 1024)
    p = engine.SearchParams(length=L, seed=5, alpha1=4, alpha2=a2, ls_lmt=3, flip_lmt=10,
                            n_lmt=n, stop=engine.StopCondition(max_nse=max_nse))
    out, best = run_chain(p, walks, rounds)
    prev = None
    chain_best = None
    for r in out:
        for w, rec in enumerate(r.records):
            rc, o, osol, oev, _ = O.run_search(L, r.seeds[w], 4, a2, 3, 10, n, max_nse,
                                               init=prev, traces_cap=0)
            assert rc == 0
            assert (rec.nse, rec.psl_best) == (o.nse, o.psl_best), (r.round, w)
            assert np.array_equal(rec.solution_best, osol), (r.round, w)
        rb = min(x.psl_best for x in r.records)
        chain_best = rb if chain_best is None else min(chain_best, rb)
        assert r.chain_best_psl == chain_best and r.round_best_psl == rb
        i = r.round_best_walk
        if prev is None or r.records[i].psl_best < O.psl(O.build_table(prev)):
            prev = r.records[i].solution_best.copy()
    assert O.psl(O.build_table(best)) == out[-1].chain_best_psl
    two, best2 = run_chain(p, walks, rounds, devices=[0, 0])
    assert [x.chain_best_psl for x in two] == [x.chain_best_psl for x in out]
    assert np.array_equal(best, best2)
