"""Row-by-row proof that the certified scan's intervals hold the reference's
serial doubles at the BASELINE lengths, in both alpha regimes.

With the certificate check on (psl_ctx_set_cert_check), every step the
certified tensor-core scan scores is ALSO re-scored by the exact serial-chain
sweep (itself bit-identical to detail::eval_flip, sequence.hpp:126-162 --
test_gpu_parity.py).  The kernel then tests, for every row j of the step,
V_exact(j) in [lo(j), hi(j)], and compares the decisions the intervals took on
their own (argmin with smallest-offset ties, value_step vs value_local;
search.cpp:383-413) with the exact ones.  Decisions are taken from the exact
sweep in this mode, so the walks are the reference's walks.

The large-alpha runs put alpha2 (13 / 11 / 10 at m16 / m18 / m20,
search.cpp:19-23) into phase 1 so that regime -- terms up to ~1e37 at m20,
fixed-point scale 2^qH with qH ~ 60 -- is checked at full n_lmt = 1024 from the
first step; the n_lmt = 2, ls_lmt = 1 runs switch phase every few steps and
check the restart path (snapshot restore, 10 folded flips, serial fitness chain).
"""
import pytest

pytestmark = pytest.mark.gpu


def _run(engine, L, a1, a2, ls, n, walks, steps, seed=11):
    ctx = engine.default_context()
    ctx.set_cert_check(True)
    try:
        before = ctx.cert_check_stats()
        sb = ctx.scan_stats()
        p = engine.SearchParams(length=L, seed=seed, alpha1=a1, alpha2=a2, ls_lmt=ls,
                                flip_lmt=min(L, 10), n_lmt=n,
                                stop=engine.StopCondition(max_nse=1 + steps * (n + 1)))
        w = engine.Walks(p, walks, seeds=[seed + i for i in range(walks)], ctx=ctx)
        w.run()
        recs = w.records()
        w.close()
    finally:
        ctx.set_cert_check(False)
    after = ctx.cert_check_stats()
    sa = ctx.scan_stats()
    d = {k: after[k] - before[k] for k in ("steps", "rows", "violations", "decided",
                                         "decided_wrong")}
    d["tightness"], d["rel_width"] = after["tightness"], after["rel_width"]
    d["switches"] = sum(r.switches for r in recs)
    d["certified"] = sa["certified"] - sb["certified"]
    return d


@pytest.mark.parametrize("L,a1,a2,walks,steps", [
    (65535, 4, 13, 8, 40), (65535, 13, 4, 8, 40),
    (262143, 4, 11, 4, 16), (262143, 11, 4, 4, 16),
    (1048575, 4, 10, 3, 8), (1048575, 10, 4, 3, 8),
])
def test_intervals_hold_exact_doubles_full_neighbourhood(engine, L, a1, a2, walks, steps):
    d = _run(engine, L, a1, a2, 2000, 1024, walks, steps)
    assert d["steps"] >= walks * (steps - 1), d
    assert d["rows"] >= d["steps"] * 1024 - 1024, d
    assert d["violations"] == 0, d
    assert d["decided"] > 0 and d["decided_wrong"] == 0, d
    assert d["tightness"] <= 1.0, d


@pytest.mark.parametrize("L,a2,n,steps", [(65535, 13, 2, 400), (262143, 11, 2, 200),
                                          (1048575, 10, 2, 150)])
def test_intervals_hold_across_phase_switches(engine, L, a2, n, steps):
    d = _run(engine, L, 4, a2, 1, n, 2, steps)
    assert d["switches"] >= 4, d            # both phases, restarts included
    assert d["violations"] == 0 and d["decided_wrong"] == 0, d
    assert d["rows"] > 0 and d["decided"] > 0, d


def _deep_start(name, L):
    import json
    import os
    import numpy as np
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "phase2.json")))
    d = g[name]
    bits = np.unpackbits(np.frombuffer(bytes.fromhex(d["init_bits_hex"]), np.uint8),
                         bitorder="little")[:L]
    return np.where(bits == 1, -1, 1).astype(np.int8)


@pytest.mark.parametrize("name,L,a2,steps,walks", [("m16_deep_ls1", 65535, 13, 150, 4),
                                                  ("m18_deep_ls1", 262143, 11, 40, 3)])
def test_intervals_hold_full_neighbourhood_in_both_phases(engine, name, L, a2, steps, walks):
    """Deep warm starts (the phase2.json fixtures'), n_lmt 1024, ls_lmt 1: the walks
    switch phase, so alpha2 steps score the full neighbourhood under the check."""
    ctx = engine.default_context()
    init = _deep_start(name, L)
    ctx.set_cert_check(True)
    try:
        before = ctx.cert_check_stats()
        p = engine.SearchParams(length=L, seed=21, alpha1=4, alpha2=a2, ls_lmt=1,
                                flip_lmt=10, n_lmt=1024,
                                stop=engine.StopCondition(max_nse=1 + steps * 1024))
        w = engine.Walks(p, walks, seeds=[21 + i for i in range(walks)], inits=init, ctx=ctx)
        w.run()
        recs = w.records()
        w.close()
    finally:
        ctx.set_cert_check(False)
    after = ctx.cert_check_stats()
    assert sum(r.switches for r in recs) >= walks
    assert after["violations"] == before["violations"]
    assert after["decided_wrong"] == before["decided_wrong"]
    assert after["rows"] - before["rows"] >= walks * (steps // 2) * 1024


@pytest.mark.slow
def test_m20_auto_vs_exact_at_bench_scale(engine):
    """The benchmarked configuration (m20, 444 walks = three waves, n_lmt 1024) with
    ls_lmt 2, 50 steps: every walk's record and best sequence from the certified
    scan equals the exact sweep's (A/B at scale)."""
    import numpy as np
    ctx = engine.default_context()
    L = 1048575
    p = engine.SearchParams(length=L, seed=1, alpha1=4, alpha2=10, ls_lmt=2, flip_lmt=10,
                            n_lmt=1024, stop=engine.StopCondition(max_nse=1 + 50 * 1024))
    out = {}
    for mode in (ctx.SCAN_AUTO, ctx.SCAN_EXACT):
        ctx.set_scan_mode(mode)
        before = ctx.scan_stats()
        out[mode] = engine.run_walks(p, 444, ctx=ctx)
        after = ctx.scan_stats()
        if mode == ctx.SCAN_AUTO:
            assert after["certified"] - before["certified"] >= 444 * 45
    ctx.set_scan_mode(ctx.SCAN_AUTO)
    for a, b in zip(out[ctx.SCAN_AUTO], out[ctx.SCAN_EXACT]):
        assert (a.seed, a.nse, a.psl_best, a.energy, a.switches, a.steps) == \
            (b.seed, b.nse, b.psl_best, b.energy, b.switches, b.steps)
        assert np.array_equal(a.solution_best, b.solution_best)


@pytest.mark.parametrize("L,a1,a2", [(1048575, 4, 10), (262143, 11, 4)])
def test_forced_fallbacks_at_baseline_lengths(engine, monkeypatch, L, a1, a2):
    """Widened intervals (PSLB200_CERT_SLACK) at m20 / m18 push many steps onto the
    exact re-score and the exact value_local chain (the fallback the benchmark
    never needed at m20): the records still equal the exact sweep's."""
    import numpy as np
    ctx = engine.default_context()
    p = engine.SearchParams(length=L, seed=9, alpha1=a1, alpha2=a2, ls_lmt=2, flip_lmt=10,
                            n_lmt=1024, stop=engine.StopCondition(max_nse=1 + 6 * 1024))
    ctx.set_scan_mode(ctx.SCAN_EXACT)
    ref = engine.run_walks(p, 3, ctx=ctx)
    ctx.set_scan_mode(ctx.SCAN_AUTO)
    monkeypatch.setenv("PSLB200_CERT_SLACK", "1e-5")
    before = ctx.scan_stats()
    got = engine.run_walks(p, 3, ctx=ctx)
    after = ctx.scan_stats()
    assert after["refined"] - before["refined"] > 0
    for a, b in zip(got, ref):
        assert (a.nse, a.psl_best, a.energy) == (b.nse, b.psl_best, b.energy)
        assert np.array_equal(a.solution_best, b.solution_best)


@pytest.mark.parametrize("L,steps", [(262143, 4), (1048575, 2)])
def test_paper_neighbourhood_6912_auto_equals_exact(engine, L, steps):
    """The paper's N_lmt = 6912: seven certified 1024-row groups
    per step combined in ascending offset order; records equal the exact sweep's."""
    import numpy as np
    ctx = engine.default_context()
    p = engine.SearchParams(length=L, seed=4, alpha1=4, alpha2=engine.default_alpha2(L),
                            ls_lmt=2000, flip_lmt=10, n_lmt=6912,
                            stop=engine.StopCondition(max_nse=1 + steps * 6912))
    out = {}
    for mode in (ctx.SCAN_EXACT, ctx.SCAN_AUTO):
        ctx.set_scan_mode(mode)
        out[mode] = engine.run_walks(p, 2, ctx=ctx)
    ctx.set_scan_mode(ctx.SCAN_AUTO)
    for a, b in zip(out[ctx.SCAN_AUTO], out[ctx.SCAN_EXACT]):
        assert (a.nse, a.psl_best, a.energy, a.steps) == (b.nse, b.psl_best, b.energy, b.steps)
        assert np.array_equal(a.solution_best, b.solution_best)
