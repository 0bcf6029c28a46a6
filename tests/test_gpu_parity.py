"""Parity of the sm_100a engine (through the C ABI) with the reference.

Every comparison is bit-exact: C_k / PSL / indices as integers, fitness values
as IEEE doubles (hex).  Ground truth is the golden vectors generated from the
unmodified reference (tests/golden/) and the pinned CPU oracle (oracle/) on
seeded random inputs at sizes it finishes in seconds.
"""
import hashlib

import numpy as np
import pytest

from oracle import oracle_py as O
from util import from_pm, hx, to_pm, unhex

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ------------------------------------------------------------------ tables

@pytest.mark.parametrize("L", [2, 3, 4, 5, 31, 32, 33, 127, 128, 129, 1000, 4095, 4096, 4097,
                               16383, 65535])
def test_build_table_matches_oracle(engine, L):
    rng = np.random.default_rng(L)
    s = rng.choice(np.array([-1, 1], np.int8), L)
    got = engine.build_table(s)
    assert got[0] == L
    assert np.array_equal(got, O.build_table(s, fast=True))


def test_build_table_golden(engine, golden):
    g = golden("hand.json")
    assert list(engine.build_table(np.ones(4, np.int8))) == g["ones4_table"]
    assert list(engine.build_table(np.array([1, -1, 1, -1], np.int8))) == g["alt4_table"]
    b13 = np.array([1, 1, 1, 1, 1, -1, -1, 1, 1, -1, 1, -1, 1], np.int8)
    t = engine.build_table(b13)
    assert list(t) == g["barker13_table"]
    assert engine.psl(t) == 1 and engine.merit_factor(t) == 169.0 / 12.0


def test_build_table_kats(engine, golden):
    for L, g in golden("kats.json").items():
        s = O.random_sequence(1, int(L))
        assert sha(engine.build_table(s)) == g["table_sha"]


def test_apply_flip_matches_oracle(engine):
    rng = np.random.default_rng(5)
    for L in (2, 3, 17, 64, 65, 300, 5000):
        s = rng.choice(np.array([-1, 1], np.int8), L)
        c = O.build_table(s)
        for _ in range(4):
            j = int(rng.integers(0, L))
            s2, c2 = s.copy(), c.copy()
            engine.apply_flip(s, c, j)
            O.apply_flip(s2, c2, j)
            assert np.array_equal(s, s2) and np.array_equal(c, c2)
        assert np.array_equal(c, O.build_table(s))


# ------------------------------------------------------------------ scans

def test_scan_golden_vectors(engine, golden):
    for case in golden("scans.json"):
        L = case["L"]
        s = O.random_sequence(case["seed"], L)
        c = O.build_table(s, fast=True)
        lut = O.power_table(L, case["alpha"])
        v, p = engine.scan_values(s, c, case["start"], case["n"], lut)
        assert sha(v[1:]) == case["values_sha"], (L, case["n"])
        assert sha(p[1:]) == case["psls_sha"], (L, case["n"])
        if "values" in case:
            assert [hx(x) for x in v[1:]] == case["values"]
        r = engine.neighborhood_scan(s, c, engine.PowerTable(L, case["alpha"]), case["start"],
                                     case["n"])
        assert (r.best_index, hx(r.value_step), r.best_neighbor_psl, r.best_psl_index) == \
            (case["best_index"], case["value_step"], case["best_neighbor_psl"],
             case["best_psl_index"])


def test_scan_random_vs_oracle(engine):
    rng = np.random.default_rng(2025)
    for _ in range(30):
        L = int(rng.choice([2, 3, 7, 50, 97, 500, 1023, 1500, 3000, 8191, 20000]))
        s = rng.choice(np.array([-1, 1], np.int8), L)
        c = O.build_table(s, fast=True)
        alpha = int(rng.integers(1, 14))
        lut = O.power_table(L + 4, alpha)
        start = int(rng.integers(0, L))
        n = int(rng.integers(1, min(L, 2500) + 1))
        v, p = engine.scan_values(s, c, start, n, lut)
        vo, po = O.scan(s, c, start, n, lut)
        assert np.array_equal(v.view(np.uint64)[1:], vo.view(np.uint64)[1:]), (L, start, n)
        assert np.array_equal(p[1:], po[1:]), (L, start, n)


def test_scan_full_neighbourhood_wraps(engine):
    # n == L at small L: every warp contains the (start + i) % L wrap
    for L in (33, 64, 100, 1024, 1025, 2047):
        s = O.random_sequence(L, L)
        c = O.build_table(s)
        lut = O.power_table(L, 4)
        for start in (0, L // 2, L - 1):
            v, p = engine.scan_values(s, c, start, L, lut)
            vo, po = O.scan(s, c, start, L, lut)
            assert np.array_equal(v.view(np.uint64)[1:], vo.view(np.uint64)[1:])
            assert np.array_equal(p[1:], po[1:])


def test_tie_break(engine, golden):
    ones = np.ones(4, np.int8)
    t = engine.build_table(ones)
    for case in golden("hand.json")["ones4_scans"]:
        r = engine.neighborhood_scan(ones, t, engine.PowerTable(5, case["alpha"]), case["start"],
                                     case["n"])
        assert r.best_index == case["best_index"]
        assert r.best_psl_index == case["best_psl_index"]
        assert hx(r.value_step) == case["value_step"]
        assert r.best_neighbor_psl == case["best_neighbor_psl"]
    with pytest.raises(engine.ConfigError):
        engine.neighborhood_scan(ones, t, engine.PowerTable(5, 2), 4, 4)
    with pytest.raises(engine.ConfigError):
        engine.neighborhood_scan(ones, t, engine.PowerTable(5, 2), 0, 5)


def test_c1_evaluate_neighbor(engine, golden):
    """acceptance.cpp:75-99 (C1): 1000 triples, seed 20250816, bit for bit."""
    import ctypes as C
    r = O.OrcRng()
    O.lib().orc_rng_seed(C.byref(r), 20250816)
    for (L, j, alpha, fit, psl) in golden("c1.json"):
        s = np.array([1 if (O.lib().orc_rng_next(C.byref(r)) >> 63) == 0 else -1
                      for _ in range(L)], np.int8)
        assert O.lib().orc_rng_bounded(C.byref(r), L) == j
        assert 1 + O.lib().orc_rng_bounded(C.byref(r), 13) == alpha
        t = O.build_table(s)
        e = engine.evaluate_neighbor(s, t, j, alpha)
        assert hx(e.fitness) == fit and e.psl == psl


def test_overflow_in_scan_raises(engine):
    s = np.ones(64, np.int8)
    t = engine.build_table(s)
    with pytest.raises(engine.OverflowError):
        engine.evaluate_neighbor(s, t, 5, engine.PowerTable(64, 1100))


# ------------------------------------------------------------------ run_search

def _params(engine, L, seed, a1, a2, ls, flip, n, max_nse, init=None):
    return engine.SearchParams(length=L, seed=seed, alpha1=a1, alpha2=a2, ls_lmt=ls,
                               flip_lmt=flip, n_lmt=n, stop=engine.StopCondition(max_nse=max_nse),
                               init=init)


def _run_and_compare(engine, g, with_traces=True, trace_prefix=None):
    init = from_pm(g["init"]) if "init" in g else None
    p = _params(engine, *g["params"][:8], init=init)
    traces = []
    hooks = engine.SearchHooks(on_scan=traces.append) if with_traces else None
    if g["status"] != 0:
        exc = engine.OverflowError if g["status"] == 2 else engine.ConfigError
        events = []
        with pytest.raises(exc) as ei:
            engine.run_search(p, engine.SearchHooks(on_event=events.append))
        assert str(ei.value) == g["error"]
        assert [[e.nse, e.psl_best, e.phase_index, int(e.kind)] for e in events] == g["events"]
        return
    rec = engine.run_search(p, hooks)
    assert rec.nse == g["nse"]
    assert rec.psl_best == g["psl_best"]
    assert hx(rec.merit_factor) == g["merit_factor"]
    assert to_pm(rec.solution_best) == g["solution_best"]
    assert [[e.nse, e.psl_best, e.phase_index, int(e.kind)] for e in rec.events] == g["events"]
    assert rec.solver_version == "0.1.0"
    if with_traces and "traces" in g:
        got = [[t.nse, hx(t.value_step), hx(t.value_local), t.psl_best, t.phase_index]
               for t in traces]
        assert got == g["traces"]
    return rec, traces


def test_trajectories_bit_for_bit(engine, golden):
    """unit_search.cpp:173-227: run_search == the naive reference trajectory."""
    for g in golden("trajectories.json"):
        _run_and_compare(engine, g)


def test_golden_record_formats_md(engine, golden):
    g = golden("records.json")["formats_md"]
    rec, _ = _run_and_compare(engine, g)
    assert rec.merit_factor == 4.571428571428571
    assert len(rec.events) == 4


def test_warm_start_and_overflow(engine, golden):
    g = golden("records.json")
    for key in ("warm_start_nse1", "warm_start_200", "overflow_alpha2", "overflow_alpha1"):
        _run_and_compare(engine, g[key])


def test_c6_record(engine, golden):
    """acceptance.cpp:232-254 configuration: L=4095, seed 1, 1e6 NSE."""
    g = golden("records.json")["c6"]
    p = _params(engine, *g["params"][:8])
    traces = []
    rec = engine.run_search(p, engine.SearchHooks(on_scan=traces.append))
    assert (rec.nse, rec.psl_best) == (g["nse"], g["psl_best"]) == (1000449, 57)
    assert hx(rec.merit_factor) == g["merit_factor"]
    assert to_pm(rec.solution_best) == g["solution_best"]
    assert [[e.nse, e.psl_best, e.phase_index, int(e.kind)] for e in rec.events] == g["events"]
    got = [[t.nse, hx(t.value_step), hx(t.value_local), t.psl_best, t.phase_index] for t in traces]
    assert len(got) == g["n_traces"]
    assert got[:50] == g["traces_head"]
    import json
    assert hashlib.sha256(json.dumps(got).encode()).hexdigest() == g["traces_sha"]


@pytest.mark.parametrize("L", ["16383", "65535"])
def test_kat_runs(engine, golden, L):
    g = golden("kats.json")[L]
    _run_and_compare(engine, g)


@pytest.mark.parametrize("L", ["262143", "1048575"])
def test_kat_runs_big(engine, golden, L):
    g = golden("kats_big.json")[L]
    _run_and_compare(engine, g)


def test_random_runs_vs_oracle(engine):
    rng = np.random.default_rng(77)
    for _ in range(12):
        L = int(rng.integers(2, 300))
        seed = int(rng.integers(1, 1 << 40))
        a1, a2 = int(rng.integers(1, 8)), int(rng.integers(1, 14))
        ls, flip = int(rng.integers(1, 6)), int(rng.integers(1, L + 1))
        n = int(rng.integers(1, L + 1))
        max_nse = int(rng.integers(1, 20000))
        rc, rec, sol, ev, tr = O.run_search(L, seed, a1, a2, ls, flip, n, max_nse,
                                            traces_cap=1 << 16)
        traces = []
        p = _params(engine, L, seed, a1, a2, ls, flip, n, max_nse)
        if rc != 0:
            with pytest.raises(engine.OverflowError):
                engine.run_search(p)
            continue
        r = engine.run_search(p, engine.SearchHooks(on_scan=traces.append))
        assert (r.nse, r.psl_best, to_pm(r.solution_best)) == (rec.nse, rec.psl_best, to_pm(sol))
        assert hx(r.merit_factor) == hx(rec.merit_factor)
        assert [(e.nse, e.psl_best, e.phase_index, int(e.kind)) for e in r.events] == ev
        assert [(t.nse, t.value_step, t.value_local, t.psl_best, t.phase_index)
                for t in traces] == tr


def test_large_neighbourhood_groups(engine):
    """n_lmt > 1024 (paper's 6912-style): several 1024-neighbour groups per step."""
    L, n = 5000, 3000
    rc, rec, sol, ev, tr = O.run_search(L, 9, 4, 13, 3, 10, n, 1 + 12 * n, traces_cap=64)
    assert rc == 0
    traces = []
    r = engine.run_search(_params(engine, L, 9, 4, 13, 3, 10, n, 1 + 12 * n),
                          engine.SearchHooks(on_scan=traces.append))
    assert [(t.nse, t.value_step, t.value_local, t.psl_best, t.phase_index) for t in traces] == tr
    assert r.psl_best == rec.psl_best and to_pm(r.solution_best) == to_pm(sol)


# ------------------------------------------------------------------ many walks

def test_walks_equal_single_runs(engine):
    """Walk independence: walk w of a batch == run_search(seed0 + w)."""
    L, n_walks = 777, 5
    p = _params(engine, L, 100, 4, 13, 20, 10, 300, 1 + 60 * 300)
    recs = engine.run_walks(p, n_walks)
    for w, r in enumerate(recs):
        q = _params(engine, L, 100 + w, 4, 13, 20, 10, 300, 1 + 60 * 300)
        single = engine.run_search(q)
        assert (r.nse, r.psl_best) == (single.nse, single.psl_best)
        assert np.array_equal(r.solution_best, single.solution_best)
        assert r.merit_factor == single.merit_factor


def test_walks_full_size_properties(engine):
    """At the headline length: solution_best re-verifies to psl_best and the
    record's merit factor (device int64 energy) matches a fresh table build."""
    L = 1048575
    p = engine.SearchParams(length=L, seed=1, alpha1=4, alpha2=10, ls_lmt=2000, flip_lmt=10,
                            n_lmt=1024, stop=engine.StopCondition(max_nse=1 + 3 * 1024))
    w = engine.Walks(p, 2)
    w.run()
    recs = w.records(solutions=True)
    w.close()
    kat = None
    try:
        from conftest import load_golden
        kat = load_golden("kats_big.json")["1048575"]
    except BaseException:
        pass
    for r in recs:
        t = engine.build_table(r.solution_best)
        assert engine.psl(t) == r.psl_best
        assert engine.merit_factor(t) == r.merit_factor
        assert r.nse == 1 + 3 * 1024
    if kat:
        assert recs[0].psl_best == kat["psl_best"]
        assert to_pm(recs[0].solution_best) == kat["solution_best"]
        assert hx(recs[0].merit_factor) == kat["merit_factor"]


def test_max_seconds_stop(engine):
    p = engine.SearchParams(length=256, seed=4, stop=engine.StopCondition(max_seconds=0.05))
    rec = engine.run_search(p)
    assert rec.nse > 1
    assert rec.elapsed_seconds >= 0.05
    assert rec.elapsed_seconds < 5.0


def test_walks_warm_starts(engine):
    """Per-walk warm starts (validated and packed on the device) == run_search(init)."""
    L = 300
    rng = np.random.default_rng(8)
    inits = np.where(rng.integers(0, 2, (3, L)) == 1, -1, 1).astype(np.int8)
    p = _params(engine, L, 5, 4, 13, 6, 10, 100, 1 + 40 * 100)
    recs = engine.run_walks(p, 3, inits=inits)
    for w, r in enumerate(recs):
        q = _params(engine, L, 5 + w, 4, 13, 6, 10, 100, 1 + 40 * 100, init=inits[w])
        single = engine.run_search(q)
        rc, orec, osol, _, _ = O.run_search(L, 5 + w, 4, 13, 6, 10, 100, 1 + 40 * 100,
                                            init=inits[w])
        assert (r.nse, r.psl_best) == (single.nse, single.psl_best) == (orec.nse, orec.psl_best)
        assert np.array_equal(r.solution_best, osol)
    bad = inits.copy()
    bad[1, 17] = 0
    with pytest.raises(engine.ConfigError, match="position 17 is 0"):
        engine.run_walks(p, 3, inits=bad)


def test_walks_warm_starts_unaligned(engine):
    """Odd L: walks start at every byte alignment of the packed-int8 upload
    (the device validates / packs 32-byte groups with aligned loads + funnel
    shifts); first offending element wins."""
    L, nw = 301, 6
    rng = np.random.default_rng(9)
    inits = np.where(rng.integers(0, 2, (nw, L)) == 1, -1, 1).astype(np.int8)
    p = _params(engine, L, 11, 4, 13, 6, 10, 64, 1 + 8 * 64)
    recs = engine.run_walks(p, nw, inits=inits)
    for w, r in enumerate(recs):
        rc, orec, osol, _, _ = O.run_search(L, 11 + w, 4, 13, 6, 10, 64, 1 + 8 * 64, init=inits[w])
        assert (r.nse, r.psl_best) == (orec.nse, orec.psl_best)
        assert np.array_equal(r.solution_best, osol)
    for (w, i, v) in ((3, 40, 2), (5, 300, 0), (1, 63, -3)):
        bad = inits.copy()
        bad[w, i] = v
        if i + 100 < L:
            bad[w, i + 100] = 7            # a later offender in the same walk is not reported
        with pytest.raises(engine.ConfigError, match=f"position {i} is {v};"):
            engine.run_walks(p, nw, inits=bad)


def test_walks_warm_starts_batched_upload(engine):
    """Many long warm-started walks: uploaded in four batches on a copy stream,
    each batch packed and its NTT tables built while the next one is in flight."""
    L, nw = 9001, 40
    rng = np.random.default_rng(12)
    inits = np.where(rng.integers(0, 2, (nw, L)) == 1, -1, 1).astype(np.int8)
    p = _params(engine, L, 30, 4, 13, 3, 10, 256, 1 + 4 * 256)
    recs = engine.run_walks(p, nw, inits=inits)
    for w in (0, 9, 10, 19, 20, 30, 39):          # first / last walk of each batch
        rc, orec, osol, _, _ = O.run_search(L, 30 + w, 4, 13, 3, 10, 256, 1 + 4 * 256, init=inits[w])
        assert (recs[w].nse, recs[w].psl_best) == (orec.nse, orec.psl_best)
        assert np.array_equal(recs[w].solution_best, osol)
    bad = inits.copy()
    bad[37, 4000] = 3
    bad[38, 5] = 0                                 # a later walk: not the first offender
    with pytest.raises(engine.ConfigError, match="position 4000 is 3;"):
        engine.run_walks(p, nw, inits=bad)


@pytest.mark.parametrize("L", [8192, 8193, 16385, 40000, 131073, 262145])
def test_ntt_table_build_lengths(engine, L):
    """Walk tables of every four-step shape (R x C = 128x128 .. 512x1024, the
    radix-8 rounds with a 1- or 2-stage remainder) against the oracle: the
    first steps, the PSL and the merit factor (exact energy over all C_k)."""
    nw = 2
    rng = np.random.default_rng(L)
    inits = np.where(rng.integers(0, 2, (nw, L)) == 1, -1, 1).astype(np.int8)
    p = _params(engine, L, 50, 4, 13, 3, 10, 64, 1 + 2 * 64)
    recs = engine.run_walks(p, nw, inits=inits)
    for w in range(nw):
        rc, orec, osol, _, _ = O.run_search(L, 50 + w, 4, 13, 3, 10, 64, 1 + 2 * 64, init=inits[w])
        assert (recs[w].nse, recs[w].psl_best) == (orec.nse, orec.psl_best)
        assert hx(recs[w].merit_factor) == hx(orec.merit_factor)
        assert np.array_equal(recs[w].solution_best, osol)


def test_run_walks_pinned_solutions(engine):
    """psl_run_walks into a pinned buffer: the run kernel writes every walk's
    best sequence over PCIe as the walk stops (odd L: unaligned rows, head and
    tail bytes); equal to the unpack + D2H path and to the oracle."""
    import torch
    for L, nw in ((9001, 5), (4097, 3), (70001, 2)):
        p = _params(engine, L, 11, 4, 13, 3, 10, 128, 1 + 3 * 128)
        pinned = torch.full((nw, L), 7, dtype=torch.int8).pin_memory().numpy()
        r1 = engine.run_walks(p, nw, out=pinned)
        r2 = engine.run_walks(p, nw)
        w = engine.Walks(p, nw)
        w.run()
        r3 = w.records(solutions=True)
        w.close()
        for a, b, c in zip(r1, r2, r3):
            assert (a.nse, a.psl_best, a.energy) == (b.nse, b.psl_best, b.energy) == (c.nse, c.psl_best, c.energy)
            assert np.array_equal(a.solution_best, b.solution_best)
            assert np.array_equal(a.solution_best, c.solution_best)
        rc, orec, osol, _, _ = O.run_search(L, 11, 4, 13, 3, 10, 128, 1 + 3 * 128)
        assert np.array_equal(pinned[0], osol) and r1[0].psl_best == orec.psl_best


def test_drain_and_resume(engine, golden, monkeypatch):
    """Tiny device event/trace buffers: run_search drains and relaunches many
    times; hooks must still see the reference's exact event/trace stream."""
    monkeypatch.setenv("PSLB200_DRAIN_CAP", "3")
    for key in ("formats_md", "warm_start_200"):
        _run_and_compare(engine, golden("records.json")[key])
    for g in golden("trajectories.json")[:3]:
        _run_and_compare(engine, g)


def test_verify_sequence_matches_oracle(engine):
    """oracle::verify_sequence on the device: PSL, merit factor, histogram."""
    rng = np.random.default_rng(12)
    for L in (2, 13, 100, 4097, 70000):
        s = rng.choice(np.array([-1, 1], np.int8), L)
        c = O.build_table(s, fast=True)
        rep = engine.verify_sequence(s)
        assert rep.psl == O.psl(c)
        assert rep.merit_factor == O.lib().orc_merit_factor(c, L)
        hist = np.bincount(np.abs(c[1:]), minlength=rep.psl + 1)
        assert np.array_equal(rep.sidelobe_histogram, hist)
