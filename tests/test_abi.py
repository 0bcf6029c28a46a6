"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every entry point include/pslb200.h declares, and its host logic (defaults,
validation, pow_int, error classes) matches the reference (search.cpp:19-94,
sequence.cpp:95-105, unit_search.cpp:34-103).  No compute call needs a GPU here;
without one, compute entry points must fail loudly (no CPU fallback)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2107_09801_b200 as P
from paper_2107_09801_b200 import _lib as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "pslb200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(psl_\w+)\s*\(", text, flags=re.M)
    return sorted(set(n for n in names if not n.endswith("_cb")))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(B.SO_PATH)
    declared = header_functions()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in include/pslb200.h but not exported"
    # and the Python binding covers the same surface
    assert set(declared) == set(B.SIGNATURES), set(declared) ^ set(B.SIGNATURES)


def test_version_echo():
    assert B.lib().psl_version() == b"0.1.0"          # version.hpp:5
    assert P.kVersion == "0.1.0"


def test_defaults_follow_reference():
    # unit_search.cpp:34-57
    assert [P.default_alpha2(L) for L in (1023, 16383, 131071, 262142, 262143, 524286, 524287,
                                          1048575)] == [13, 13, 13, 13, 11, 11, 10, 10]
    assert [P.default_n_lmt(L) for L in (100, 1024, 65535)] == [100, 1024, 1024]
    assert [P.default_flip_lmt(L) for L in (8, 1023)] == [8, 10]
    p = P.default_params(16383)
    assert (p.alpha1, p.alpha2, p.ls_lmt, p.flip_lmt, p.n_lmt) == (4, 13, 2000, 10, 1024)
    c = B.psl_params()
    B.lib().psl_default_params(16383, C.byref(c))
    assert (c.alpha1, c.alpha2, c.ls_lmt, c.flip_lmt, c.n_lmt, c.workers) == (4, 13, 2000, 10, 1024, 1)


def _ok(**kw):
    return P.SearchParams(length=64, seed=1, stop=P.StopCondition(max_nse=1000), **kw)


def test_validate_rejects_bad_configurations():
    # unit_search.cpp:59-89
    P.validate_params(_ok())
    bad = [dict(length=1), dict(alpha1=0), dict(ls_lmt=0), dict(workers=0), dict(flip_lmt=0),
           dict(n_lmt=0), dict(length=(1 << 20) + 1), dict(workers=5000)]
    for kw in bad:
        p = _ok()
        for k, v in kw.items():
            setattr(p, k, v)
        with pytest.raises(P.ConfigError):
            P.validate_params(p)
    p = _ok()
    p.stop = P.StopCondition()
    with pytest.raises(P.ConfigError, match="stop condition"):
        P.validate_params(p)
    p.stop = P.StopCondition(max_seconds=-1.0)
    with pytest.raises(P.ConfigError):
        P.validate_params(p)
    p = _ok(init=np.ones(63, np.int8))
    with pytest.raises(P.ConfigError, match="warm-start sequence has length 63, expected 64"):
        P.validate_params(p)
    # search.cpp:40-76 order: a bad exponent is reported before the init length
    p = _ok(init=np.ones(63, np.int8))
    p.alpha1 = 0
    with pytest.raises(P.ConfigError, match="alpha1"):
        P.validate_params(p)
    # every entry that takes params checks the length before the C ABI reads `length` bytes
    with pytest.raises(P.ConfigError, match="has length 65, expected 64"):
        P.run_search(_ok(init=np.ones(65, np.int8)))
    p = _ok(init=np.array([1, 2] * 32, np.int8))
    with pytest.raises(P.ConfigError, match="must be \\+1 or -1"):
        P.validate_params(p)


def test_validate_clamps_with_warning():
    # unit_search.cpp:91-103
    p = P.SearchParams(length=16, n_lmt=1024, flip_lmt=100, stop=P.StopCondition(max_nse=1000))
    warn = []
    q = P.validate_params(p, warn)
    assert (q.n_lmt, q.flip_lmt) == (16, 16)
    assert "n-lmt" in warn[0] and "flip-lmt" in warn[0]


def test_pow_int_matches_reference_kats(golden):
    g = golden("hand.json")["pow_int"]
    for a, vals in g.items():
        for alpha, v in enumerate(vals):
            assert float(B.lib().psl_pow_int(float(a), alpha)).hex() == v
    # PowerTable == pow_int entry by entry (unit_sequence.cpp:85-99)
    for alpha in (1, 2, 3, 4, 7, 13):
        lut = P.PowerTable(100, alpha)
        assert all(lut[a] == P.pow_int(float(a), alpha) for a in range(101))
    big = P.PowerTable(5000, 10)  # vectorised path, same factor order
    assert all(big[a] == P.pow_int(float(a), 10) for a in range(0, 5001, 37))


def test_host_psl_mf_and_device_only_fitness(golden):
    from oracle import oracle_py as O
    rng = np.random.default_rng(4)
    for _ in range(10):
        L = int(rng.integers(2, 300))
        s = rng.choice(np.array([-1, 1], np.int8), L)
        c = O.build_table(s)
        assert P.psl(c) == O.psl(c)
        assert P.merit_factor(c) == O.lib().orc_merit_factor(c, L)


def test_event_kinds():
    assert [P.pslopt.to_string(k) for k in P.EventKind] == ["improved-psl", "phase-switch",
                                                            "local-best-improved"]
    assert P.pslopt.event_kind_from_string("phase-switch") == P.EventKind.kPhaseSwitch
    with pytest.raises(P.ParseError):
        P.pslopt.event_kind_from_string("nope")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback_without_gpu():
    with pytest.raises(P.DeviceError, match="no CPU fallback"):
        P.Context(0)


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure mode")
def test_public_entry_points_fail_loudly_without_gpu():
    """run_walks (one psl_run_walks call), Walks and run_search: every compute
    entry raises DeviceError on a host without a B200 -- no CPU fallback."""
    L = 64
    p = P.SearchParams(length=L, seed=1, alpha1=4, alpha2=13, ls_lmt=3, flip_lmt=2, n_lmt=8,
                       stop=P.StopCondition(max_nse=100))
    with pytest.raises(P.DeviceError):
        P.run_walks(p, 2)
    with pytest.raises(P.DeviceError):
        P.Walks(p, 2)
    with pytest.raises(P.DeviceError):
        P.run_search(p)
    # fitness() / flip_deltas() run on the device (psl_fitness, psl_flip_deltas)
    c = np.zeros(L, np.int32)
    with pytest.raises(P.DeviceError):
        P.fitness(c, 4)
    with pytest.raises(P.DeviceError):
        P.flip_deltas(np.ones(L, np.int8), 0)
    with pytest.raises(P.DeviceError):
        P.run_walks_multi(p, 2, devices=[0])


def test_walk_inputs_are_size_checked_before_the_abi():
    """psl_walks_create / psl_run_walks read 8 n_walks seed bytes and
    n_walks x L start bytes: wrong sizes must raise ConfigError on the host
    (before any device or C-ABI call), one (L,) start is given to every walk."""
    p = _ok()
    with pytest.raises(P.ConfigError, match="seeds"):
        P.Walks(p, 4, seeds=[1, 2, 3])
    with pytest.raises(P.ConfigError, match="warm starts"):
        P.run_walks(p, 4, inits=np.ones((3, 64), np.int8))
    with pytest.raises(P.ConfigError, match="warm starts"):
        P.Walks(p, 2, inits=np.ones(63, np.int8))
    with pytest.raises(P.ConfigError, match="n_walks"):
        P.run_walks(p, 0)
    from paper_2107_09801_b200.pslopt import _walk_inputs
    s, i = _walk_inputs(p, 3, [5, 6, 7], np.ones(64, np.int8))
    assert s.tolist() == [5, 6, 7] and i.shape == (3, 64) and i.flags.c_contiguous


def test_scan_seam_rejects_short_power_table():
    """psl_scan reads PowerTable(L, alpha) (L + 1 entries, search.cpp:337-338): a
    shorter table is a ConfigError before any device work (no GPU needed)."""
    L = 64
    s = np.ones(L, np.int8)
    t = np.arange(L, 0, -1).astype(np.int32)
    lut = np.ones(L, np.float64)
    values, psls = np.zeros(9, np.float64), np.zeros(9, np.int32)
    job = B.psl_scan_job(s.ctypes.data, t.ctypes.data, L, 0, 8, lut.ctypes.data, len(lut),
                         values.ctypes.data, psls.ctypes.data)
    err = C.create_string_buffer(256)
    rc = B.lib().psl_scan(None, C.byref(job), err, 256)       # checked before any device use
    assert rc == B.PSL_ERR_CONFIG and b"power table too small" in err.value
