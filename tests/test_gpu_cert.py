"""The certified (decision-exact) scan: runs without an on_scan hook score
most steps with the tensor-core interval scan and fall back to the exact
sweep whenever the intervals cannot decide.  Every record, event list and
best sequence must still equal the reference's: checked here against the
golden fixtures of the unmodified reference, the pinned CPU oracle, and the
exact-sweep engine, with the fallbacks forced on (PSLB200_CERT_SLACK widens
every interval) as well as in their natural (rare) occurrence.
"""
import numpy as np
import pytest

from oracle import oracle_py as O
from util import from_pm, hx, to_pm

pytestmark = pytest.mark.gpu


def _params(engine, L, seed, a1, a2, ls, flip, n, max_nse, init=None):
    return engine.SearchParams(length=L, seed=seed, alpha1=a1, alpha2=a2, ls_lmt=ls,
                               flip_lmt=flip, n_lmt=n, stop=engine.StopCondition(max_nse=max_nse),
                               init=init)


def _stats_delta(ctx, before):
    after = ctx.scan_stats()
    return {k: after[k] - before[k] for k in after}


def _check_record(engine, g):
    init = from_pm(g["init"]) if "init" in g else None
    ctx = engine.default_context()
    before = ctx.scan_stats()
    rec = engine.run_search(_params(engine, *g["params"][:8], init=init))   # no hooks: certified
    assert rec.nse == g["nse"]
    assert rec.psl_best == g["psl_best"]
    assert hx(rec.merit_factor) == g["merit_factor"]
    assert to_pm(rec.solution_best) == g["solution_best"]
    assert [[e.nse, e.psl_best, e.phase_index, int(e.kind)] for e in rec.events] == g["events"]
    return _stats_delta(ctx, before)


@pytest.mark.parametrize("name,key", [("kats.json", "16383"), ("kats.json", "65535"),
                                      ("kats_big.json", "262143"), ("kats_big.json", "1048575"),
                                      ("records.json", "c6")])
def test_certified_runs_match_golden(engine, golden, name, key):
    st = _check_record(engine, golden(name)[key])
    assert st["certified"] > 0          # the certified scan actually scored steps


@pytest.mark.parametrize("slack", ["1e-9", "1e-7", "1e-5"])
def test_forced_fallbacks_match_golden(engine, golden, monkeypatch, slack):
    """Widened intervals: many steps take the exact re-score and the exact
    value_local chain; the record is still the reference's."""
    monkeypatch.setenv("PSLB200_CERT_SLACK", slack)
    st = _check_record(engine, golden("records.json")["c6"])
    if slack != "1e-9":
        assert st["refined"] > 0


def test_forced_fallbacks_use_chains(engine, golden, monkeypatch):
    total = {"certified": 0, "refined": 0, "chains": 0}
    for slack in ("1e-5", "1e-4", "1e-3"):
        monkeypatch.setenv("PSLB200_CERT_SLACK", slack)
        st = _check_record(engine, golden("records.json")["c6"])
        for k in total:
            total[k] += st[k]
    assert total["refined"] > 0 and total["chains"] > 0 and total["certified"] > 0


@pytest.mark.parametrize("L,n,a2,ls", [(2048, 1024, 13, 3), (5000, 1024, 7, 2), (5000, 700, 13, 4),
                                        (8191, 1024, 10, 3), (12000, 333, 13, 2)])
def test_certified_vs_oracle_with_phase_switches(engine, L, n, a2, ls):
    """Small ls_lmt: restarts, alpha2 phases and value_local resets under the
    certified scan, against the CPU oracle's run_search."""
    max_nse = 1 + 60 * n
    rc, rec, sol, ev, _ = O.run_search(L, 5, 4, a2, ls, 10, n, max_nse, traces_cap=0)
    assert rc == 0
    ctx = engine.default_context()
    before = ctx.scan_stats()
    r = engine.run_search(_params(engine, L, 5, 4, a2, ls, 10, n, max_nse))
    st = _stats_delta(ctx, before)
    assert (r.nse, r.psl_best, to_pm(r.solution_best)) == (rec.nse, rec.psl_best, to_pm(sol))
    assert hx(r.merit_factor) == hx(rec.merit_factor)
    assert [(e.nse, e.psl_best, e.phase_index, int(e.kind)) for e in r.events] == ev
    assert st["certified"] > 0


@pytest.mark.parametrize("L,n,ls,slack", [(5000, 3000, 3, None), (4097, 4097, 2, None),
                                           (9000, 2049, 4, "1e-5"), (6000, 6000, 3, "1e-4")])
def test_certified_row_groups_vs_oracle(engine, monkeypatch, L, n, ls, slack):
    """n_lmt > 1024 (the paper's N_lmt = 6912 style): one certified pass per
    group of 1024 rows, groups combined in offset order, wrapped windows inside
    groups; with widened intervals the multi-group exact re-score and value_local
    chains run too."""
    if slack:
        monkeypatch.setenv("PSLB200_CERT_SLACK", slack)
    max_nse = 1 + 25 * n
    rc, rec, sol, ev, _ = O.run_search(L, 3, 4, 13, ls, 10, n, max_nse, traces_cap=0)
    assert rc == 0
    ctx = engine.default_context()
    before = ctx.scan_stats()
    r = engine.run_search(_params(engine, L, 3, 4, 13, ls, 10, n, max_nse))
    st = _stats_delta(ctx, before)
    assert (r.nse, r.psl_best, to_pm(r.solution_best)) == (rec.nse, rec.psl_best, to_pm(sol))
    assert hx(r.merit_factor) == hx(rec.merit_factor)
    assert [(e.nse, e.psl_best, e.phase_index, int(e.kind)) for e in r.events] == ev
    assert st["certified"] + st["refined"] > 0
    if slack:
        assert st["refined"] > 0


def test_certified_high_psl_warm_start_vs_oracle(engine):
    """A warm start with a huge peak sidelobe (PSL > 6139): the PowerTable head
    does not fit in shared memory and the certified pass reads the global table."""
    L, n = 16383, 1024
    rng = np.random.default_rng(21)
    init = np.ones(L, np.int8)
    init[rng.choice(L, 2000, replace=False)] = -1        # C_1 ~ L - 4000: PSL ~ 12000
    max_nse = 1 + 20 * n
    rc, rec, sol, ev, _ = O.run_search(L, 7, 4, 13, 3, 10, n, max_nse, init=init, traces_cap=0)
    assert rc == 0
    ctx = engine.default_context()
    before = ctx.scan_stats()
    r = engine.run_search(_params(engine, L, 7, 4, 13, 3, 10, n, max_nse, init=init))
    st = _stats_delta(ctx, before)
    assert (r.nse, r.psl_best, to_pm(r.solution_best)) == (rec.nse, rec.psl_best, to_pm(sol))
    assert hx(r.merit_factor) == hx(rec.merit_factor)
    assert [(e.nse, e.psl_best, e.phase_index, int(e.kind)) for e in r.events] == ev
    assert st["certified"] > 0
    assert r.psl_best > 6139


@pytest.mark.parametrize("L,ls,slack", [(16383, 5, None), (65535, 3, None), (16383, 4, "1e-6")])
def test_walks_auto_equals_exact(engine, monkeypatch, L, ls, slack):
    if slack:
        monkeypatch.setenv("PSLB200_CERT_SLACK", slack)
    ctx = engine.Context(0)
    p = _params(engine, L, 11, 4, 13, ls, 10, 1024, 1 + 80 * 1024)
    try:
        ctx.set_scan_mode(ctx.SCAN_AUTO)
        a = engine.run_walks(p, 24, ctx=ctx)
        ctx.set_scan_mode(ctx.SCAN_EXACT)
        e = engine.run_walks(p, 24, ctx=ctx)
    finally:
        ctx.close()
    for x, y in zip(a, e):
        assert (x.nse, x.psl_best, x.energy, x.steps, x.switches) == \
               (y.nse, y.psl_best, y.energy, y.steps, y.switches)
        assert np.array_equal(x.solution_best, y.solution_best)


def test_scan_mode_api(engine):
    ctx = engine.Context(0)
    try:
        assert ctx.scan_mode() == ctx.SCAN_AUTO
        ctx.set_scan_mode(ctx.SCAN_EXACT)
        assert ctx.scan_mode() == ctx.SCAN_EXACT
        with pytest.raises(engine.ConfigError):
            ctx.set_scan_mode(7)
    finally:
        ctx.close()
