"""Pins the CPU oracle (oracle/psl_oracle.c) before it is trusted as the checker:
against the golden vectors generated from the unmodified reference
(tests/golden/*.json, tests/golden/make_golden.py) and, where it was built,
against the reference library itself (oracle/_ref/libpslref.so)."""
import hashlib
import json

import numpy as np
import pytest

from oracle import oracle_py as O
from util import from_pm, hx, to_pm, unhex


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_rng_golden(golden):
    g = golden("rng.json")
    # unit_rng.cpp:27-32 regression pin
    assert g["next16"]["42"][:4] == [1546998764402558742, 6990951692964543102,
                                     12544586762248559009, 17057574109182124193]
    for seed, outs in g["next16"].items():
        assert O.rng_outputs(int(seed), 16) == outs
    for seed, s in g["random_sequence64"].items():
        assert to_pm(O.random_sequence(int(seed), 64)) == s


def test_hand_tables(golden):
    g = golden("hand.json")
    assert list(O.build_table(np.ones(4, np.int8))) == g["ones4_table"] == [4, 3, 2, 1]
    alt = np.array([1, -1, 1, -1], np.int8)
    assert list(O.build_table(alt)) == g["alt4_table"]
    b13 = np.array([1, 1, 1, 1, 1, -1, -1, 1, 1, -1, 1, -1, 1], np.int8)
    c = O.build_table(b13)
    assert list(c) == g["barker13_table"]
    assert O.psl(c) == 1
    assert O.lib().orc_merit_factor(c, 13) == 169.0 / 12.0
    ones = O.build_table(np.ones(4, np.int8))
    assert O.fitness(ones, O.power_table(4, 1)) == 6.0
    assert O.fitness(ones, O.power_table(4, 2)) == 14.0
    for a, vals in g["pow_int"].items():
        for alpha, v in enumerate(vals):
            assert hx(O.lib().orc_pow_int(float(a), alpha)) == v


def test_tie_break_scan(golden):
    g = golden("hand.json")
    s = np.ones(4, np.int8)
    c = O.build_table(s)
    for case in g["ones4_scans"]:
        lut = O.power_table(5, case["alpha"])
        v, p = O.scan(s, c, case["start"], case["n"], lut)
        rc, bi, val, pm, pi = O.reduce(v, p, case["n"])
        assert rc == case["status"]
        assert (case["start"] + bi) % 4 == case["best_index"]
        assert hx(val) == case["value_step"]
        assert pm == case["best_neighbor_psl"]
        assert (case["start"] + pi) % 4 == case["best_psl_index"]


def test_scans_golden(golden):
    for case in golden("scans.json"):
        L = case["L"]
        s = O.random_sequence(case["seed"], L)
        c = O.build_table(s, fast=L > 300)
        assert sha(c) == case["table_sha"]
        lut = O.power_table(L, case["alpha"])
        v, p = O.scan(s, c, case["start"], case["n"], lut)
        assert sha(v[1:]) == case["values_sha"], L
        assert sha(p[1:]) == case["psls_sha"], L
        if "values" in case:
            assert [hx(x) for x in v[1:]] == case["values"]
            assert list(p[1:]) == case["psls"]
        rc, bi, val, pm, pi = O.reduce(v, p, case["n"])
        assert rc == case["status"]
        if rc == 0:
            assert (case["start"] + bi) % L == case["best_index"]
            assert hx(val) == case["value_step"]
            assert pm == case["best_neighbor_psl"]
            assert (case["start"] + pi) % L == case["best_psl_index"]


def test_c1_evaluate_neighbor(golden):
    for (L, j, alpha, fit, psl) in golden("c1.json"):
        pass  # sequences are regenerated from the RNG in the GPU test; here spot-check 30
    g = golden("c1.json")[:30]
    import ctypes as C
    r = O.OrcRng()
    O.lib().orc_rng_seed(C.byref(r), 20250816)
    for (L, j, alpha, fit, psl) in g:
        s = np.array([1 if (O.lib().orc_rng_next(C.byref(r)) >> 63) == 0 else -1
                      for _ in range(L)], np.int8)
        jj = O.lib().orc_rng_bounded(C.byref(r), L)
        aa = 1 + O.lib().orc_rng_bounded(C.byref(r), 13)
        assert (jj, aa) == (j, alpha)
        c = O.build_table(s)
        f, p = O.eval_flip(s, c, j, O.power_table(L, alpha))
        assert hx(f) == fit and p == psl


def _check_run(rec_g, traces_cap=1 << 16):
    L, seed, a1, a2, ls, flip, n, max_nse = rec_g["params"][:8]
    init = from_pm(rec_g["init"]) if "init" in rec_g else None
    rc, rec, sol, ev, tr = O.run_search(L, seed, a1, a2, ls, flip, n, max_nse, init=init,
                                        traces_cap=traces_cap)
    assert rc == rec_g["status"]
    # events before an error are part of the contract (hooks fired)
    assert [list(e) for e in ev] == rec_g["events"]
    if rc == 0:
        assert rec.nse == rec_g["nse"]
        assert rec.psl_best == rec_g["psl_best"]
        assert hx(rec.merit_factor) == rec_g["merit_factor"]
        assert to_pm(sol) == rec_g["solution_best"]
    return tr


def test_trajectories_golden(golden):
    for g in golden("trajectories.json"):
        tr = _check_run(g)
        want = g["traces"]
        got = [[t[0], hx(t[1]), hx(t[2]), t[3], t[4]] for t in tr]
        assert got == want[:len(got)]
        if g["status"] == 0:
            assert got == want


def test_records_golden(golden):
    g = golden("records.json")
    fm = g["formats_md"]
    assert fm["nse"] == 401 and fm["psl_best"] == 2
    assert fm["solution_best"] == "+-+-++--++-----+"          # docs/formats.md:49
    assert unhex(fm["merit_factor"]) == 4.571428571428571
    assert [e[3] for e in fm["events"]] == [0, 2, 0, 2]
    for key in ("formats_md", "warm_start_nse1", "warm_start_200", "overflow_alpha2",
                "overflow_alpha1"):
        _check_run(g[key])
    assert "1100" in g["overflow_alpha2"]["error"] and "alpha2" in g["overflow_alpha2"]["error"]


@pytest.mark.slow
def test_c6_record(golden):
    g = golden("records.json")["c6"]
    assert g["psl_best"] == 57 and g["nse"] == 1000449
    tr = _check_run(g, traces_cap=1 << 12)
    got = [[t[0], hx(t[1]), hx(t[2]), t[3], t[4]] for t in tr]
    assert got[:50] == g["traces_head"]


def test_kat_m14(golden):
    g = golden("kats.json")["16383"]
    L = 16383
    s = O.random_sequence(1, L)
    c = O.build_table(s, fast=True)
    assert sha(c) == g["table_sha"]
    assert int(np.abs(c[1:]).max()) == g["initial_psl"] == 402
    assert hx(O.fitness(c, O.power_table(L, 4))) == g["initial_fitness"]
    # a 20-scan prefix of the 300-scan known-answer run
    p = g["params"]
    rc, rec, sol, ev, tr = O.run_search(L, 1, 4, p[3], 2000, 10, 1024, 1 + 20 * 1024,
                                        traces_cap=64)
    got = [[t[0], hx(t[1]), hx(t[2]), t[3], t[4]] for t in tr]
    assert got == g["traces"][:20]


def test_fast_table_equals_direct():
    rng = np.random.default_rng(3)
    for L in (2, 3, 31, 32, 33, 63, 64, 65, 127, 128, 129, 1000, 2049):
        s = rng.choice(np.array([-1, 1], np.int8), L)
        assert np.array_equal(O.build_table(s, fast=False), O.build_table(s, fast=True))


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_oracle_vs_live_reference():
    """Random cases straight against the compiled reference library."""
    import ctypes as C
    R = O.ref()
    rng = np.random.default_rng(11)
    for _ in range(40):
        L = int(rng.integers(2, 400))
        s = rng.choice(np.array([-1, 1], np.int8), L)
        cref = np.empty(L, np.int32)
        R.ref_build_table(s, L, cref)
        c = O.build_table(s)
        assert np.array_equal(c, cref)
        alpha = int(rng.integers(1, 14))
        lut = O.power_table(L, alpha)
        start, n = int(rng.integers(0, L)), int(rng.integers(1, L + 1))
        v, p = O.scan(s, c, start, n, lut)
        vr, pr = np.zeros(n + 1), np.zeros(n + 1, np.int32)
        R.ref_scan_values(s, c, L, start, n, lut, vr, pr)
        assert np.array_equal(v.view(np.uint64), vr.view(np.uint64))
        assert np.array_equal(p, pr)


def test_fft_table_build_pinned(golden):
    """build_table_fft (the CPU baseline's O(L log L) pivot tables) equals the
    reference's SidelobeTable::build: exactly at small L, and by the reference's
    own table hash at m14 and m20 (seed 1)."""
    import hashlib
    for L in (2, 3, 13, 64, 1000, 4095):
        s = O.random_sequence(L, L)
        assert np.array_equal(O.build_table_fft(s), O.build_table(s)), L
    for name, L in (("kats.json", 16383), ("kats_big.json", 1048575)):
        c = O.build_table_fft(O.random_sequence(1, L))
        assert hashlib.sha256(c.tobytes()).hexdigest() == golden(name)[str(L)]["table_sha"]
