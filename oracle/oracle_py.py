"""ctypes face of the CPU checkers (TEST / BASELINE INFRASTRUCTURE ONLY).

Loads oracle/liboracle_psl.so (the C restatement, psl_oracle.c) and, when it
was built, oracle/_ref/libpslref.so (the unmodified reference compiled from
/root/reference sources by oracle/Makefile).  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle_psl.so")
REF_SO = os.path.join(HERE, "_ref", "libpslref.so")

_i8p = np.ctypeslib.ndpointer(np.int8, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


class OrcRng(C.Structure):
    _fields_ = [("s", C.c_uint64 * 4)]


class OrcParams(C.Structure):
    _fields_ = [("length", C.c_uint32), ("seed", C.c_uint64), ("alpha1", C.c_uint32),
                ("alpha2", C.c_uint32), ("ls_lmt", C.c_uint32), ("flip_lmt", C.c_uint32),
                ("n_lmt", C.c_uint32), ("max_nse", C.c_uint64), ("init", C.c_void_p)]


class OrcEvent(C.Structure):
    _fields_ = [("nse", C.c_uint64), ("psl_best", C.c_int32), ("phase", C.c_uint32),
                ("kind", C.c_uint32)]


class OrcTrace(C.Structure):
    _fields_ = [("nse", C.c_uint64), ("value_step", C.c_double), ("value_local", C.c_double),
                ("psl_best", C.c_int32), ("phase", C.c_uint32)]


class OrcRecord(C.Structure):
    _fields_ = [("nse", C.c_uint64), ("psl_best", C.c_int32), ("merit_factor", C.c_double),
                ("energy_best", C.c_int64), ("n_events", C.c_uint64), ("n_traces", C.c_uint64),
                ("switches", C.c_uint64)]


class RefEvent(C.Structure):
    _fields_ = [("nse", C.c_uint64), ("psl_best", C.c_int32), ("phase", C.c_uint32),
                ("kind", C.c_uint32), ("elapsed", C.c_double)]


RefTrace = OrcTrace  # identical layout


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"oracle library missing: {ORACLE_SO} (run `make -C oracle`)")
        L = C.CDLL(ORACLE_SO)
        L.orc_rng_seed.argtypes = [C.POINTER(OrcRng), C.c_uint64]
        L.orc_rng_next.argtypes = [C.POINTER(OrcRng)]
        L.orc_rng_next.restype = C.c_uint64
        L.orc_rng_bounded.argtypes = [C.POINTER(OrcRng), C.c_uint64]
        L.orc_rng_bounded.restype = C.c_uint64
        L.orc_pow_int.argtypes = [C.c_double, C.c_uint32]
        L.orc_pow_int.restype = C.c_double
        L.orc_power_table.argtypes = [C.c_uint32, C.c_uint32, _f64p]
        L.orc_build_table.argtypes = [_i8p, C.c_uint32, _i32p]
        L.orc_build_table_fast.argtypes = [_i8p, C.c_uint32, _i32p]
        L.orc_build_table_mt.argtypes = [_i8p, C.c_uint32, _i32p, C.c_uint32]
        L.orc_psl.argtypes = [_i32p, C.c_uint32]
        L.orc_psl.restype = C.c_int32
        L.orc_fitness.argtypes = [_i32p, C.c_uint32, _f64p]
        L.orc_fitness.restype = C.c_double
        L.orc_energy.argtypes = [_i32p, C.c_uint32]
        L.orc_energy.restype = C.c_int64
        L.orc_merit_factor.argtypes = [_i32p, C.c_uint32]
        L.orc_merit_factor.restype = C.c_double
        L.orc_flip_deltas.argtypes = [_i8p, C.c_uint32, C.c_uint32, _i32p]
        L.orc_eval_flip.argtypes = [_i8p, _i32p, C.c_uint32, C.c_uint32, _f64p,
                                    C.POINTER(C.c_double), C.POINTER(C.c_int32)]
        L.orc_apply_flip.argtypes = [_i8p, _i32p, C.c_uint32, C.c_uint32]
        L.orc_default_alpha2.argtypes = [C.c_uint32]
        L.orc_default_alpha2.restype = C.c_uint32
        L.orc_random_sequence.argtypes = [C.POINTER(OrcRng), C.c_uint32, _i8p]
        L.orc_flip_random_distinct.argtypes = [_i8p, _i32p, C.c_uint32, C.c_uint32,
                                               C.POINTER(OrcRng), _u8p]
        L.orc_scan.argtypes = [_i8p, _i32p, C.c_uint32, C.c_uint32, C.c_uint32, _f64p,
                               _f64p, _i32p]
        L.orc_reduce.argtypes = [_f64p, _i32p, C.c_uint32, C.POINTER(C.c_uint32),
                                 C.POINTER(C.c_double), C.POINTER(C.c_int32),
                                 C.POINTER(C.c_uint32)]
        L.orc_reduce.restype = C.c_int
        L.orc_run_search.argtypes = [C.POINTER(OrcParams), _i8p, C.POINTER(OrcRecord),
                                     C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64]
        L.orc_run_search.restype = C.c_int
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise RuntimeError(f"reference library missing: {REF_SO} (run `make -C oracle ref`)")
        R = C.CDLL(REF_SO)
        R.ref_rng.argtypes = [C.c_uint64, C.c_uint32, _u64p]
        R.ref_random_sequence.argtypes = [C.c_uint64, C.c_uint32, _i8p]
        R.ref_build_table.argtypes = [_i8p, C.c_uint32, _i32p]
        R.ref_build_table.restype = C.c_int
        R.ref_pow_int.argtypes = [C.c_double, C.c_uint32]
        R.ref_pow_int.restype = C.c_double
        R.ref_scan_values.argtypes = [_i8p, _i32p, C.c_uint32, C.c_uint32, C.c_uint32,
                                      _f64p, _f64p, _i32p]
        R.ref_neighborhood_scan.argtypes = [_i8p, C.c_uint32, C.c_uint32, C.c_uint32,
                                            C.c_uint32, C.POINTER(C.c_uint32),
                                            C.POINTER(C.c_double), C.POINTER(C.c_int32),
                                            C.POINTER(C.c_uint32), C.c_char_p, C.c_size_t]
        R.ref_neighborhood_scan.restype = C.c_int
        R.ref_evaluate_neighbor.argtypes = [_i8p, C.c_uint32, C.c_uint32, C.c_uint32,
                                            C.POINTER(C.c_double), C.POINTER(C.c_int32)]
        R.ref_evaluate_neighbor.restype = C.c_int
        R.ref_brute_fitness.argtypes = [_i8p, C.c_uint32, C.c_uint32]
        R.ref_brute_fitness.restype = C.c_double
        R.ref_run_search.argtypes = [C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint32,
                                     C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                     C.c_uint64, C.c_double, C.c_void_p, _i8p,
                                     C.POINTER(C.c_int32), C.POINTER(C.c_double),
                                     C.POINTER(C.c_uint64), C.POINTER(C.c_double),
                                     C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64),
                                     C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64),
                                     C.c_char_p, C.c_size_t]
        R.ref_run_search.restype = C.c_int
        R.ref_naive_search.argtypes = [C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint32,
                                       C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                       _i8p, C.POINTER(C.c_int32), C.POINTER(C.c_uint64),
                                       C.POINTER(C.c_uint64), C.c_void_p, C.c_uint64,
                                       C.POINTER(C.c_uint64)]
        R.ref_naive_search.restype = C.c_int
        R.ref_bench_walks.argtypes = [C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint64,
                                      C.c_uint32, C.POINTER(C.c_uint64),
                                      C.POINTER(C.c_double), C.POINTER(C.c_double)]
        R.ref_bench_walks.restype = C.c_double
        R.ref_bench_eval.argtypes = [_i8p, _i32p, C.c_uint32, C.c_uint32, _f64p, C.c_uint32,
                                     C.c_uint32, C.c_uint32, C.POINTER(C.c_double)]
        R.ref_bench_eval.restype = C.c_double
        R.ref_walks_create.argtypes = [_u64p, C.c_uint32, C.c_uint32, C.c_uint32, _i32p, _f64p]
        R.ref_walks_create.restype = C.c_void_p
        R.ref_walks_destroy.argtypes = [C.c_void_p]
        R.ref_walks_step.argtypes = [C.c_void_p, C.c_uint32, C.POINTER(C.c_double), _i32p]
        R.ref_walks_step.restype = C.c_double
        _ref = R
    return _ref


# --------------------------------------------------------------- helpers

def rng_outputs(seed: int, count: int) -> list[int]:
    r = OrcRng()
    lib().orc_rng_seed(C.byref(r), seed)
    return [lib().orc_rng_next(C.byref(r)) for _ in range(count)]


def random_sequence(seed: int, L: int) -> np.ndarray:
    r = OrcRng()
    lib().orc_rng_seed(C.byref(r), seed)
    s = np.empty(L, np.int8)
    lib().orc_random_sequence(C.byref(r), L, s)
    return s


def power_table(max_abs: int, alpha: int) -> np.ndarray:
    lut = np.empty(max_abs + 1, np.float64)
    lib().orc_power_table(max_abs, alpha, lut)
    return lut


def build_table(s: np.ndarray, fast: bool | None = None, threads: int = 0) -> np.ndarray:
    s = np.ascontiguousarray(s, np.int8)
    L = len(s)
    c = np.empty(L, np.int32)
    if fast is None:
        fast = L > 4096
    if threads > 1:
        lib().orc_build_table_mt(s, L, c, threads)
    else:
        (lib().orc_build_table_fast if fast else lib().orc_build_table)(s, L, c)
    return c


def build_table_fft(s: np.ndarray) -> np.ndarray:
    """C_k = sum_i s_i s_{i+k} (SidelobeTable::build, sequence.cpp:46-60) as a
    float64 FFT autocorrelation rounded to integers -- O(L log L) setup for the
    CPU baseline's per-thread pivots.  Exact: the rounding error is < 1e-6 for
    L <= 2^20 (checked below, with the parity invariant C_k = L - k mod 2); the
    m20 result is pinned to the reference's table hash in tests/test_oracle.py."""
    x = np.asarray(s, np.float64)
    L = len(x)
    N = 1 << (2 * L - 1).bit_length()
    X = np.fft.rfft(x, N)
    r = np.fft.irfft(X * np.conj(X), N)[:L]
    c = np.rint(r)
    if L > 1 and float(np.abs(r - c).max()) > 0.05:
        raise RuntimeError("FFT table build lost integer precision")
    c = c.astype(np.int32)
    c[0] = L
    k = np.arange(L)
    if np.any(((c[1:] - (L - k[1:])) & 1) != 0):
        raise RuntimeError("FFT table build broke the sidelobe parity invariant")
    return c


class RefWalks:
    """The reference's step loop on all host threads, one independent walk per
    thread (ref_shim.cpp ref_walks_*): walk w = run_search(seed_w)'s pivot,
    table from build_table_fft (setup, untimed)."""

    def __init__(self, seeds, L: int, n: int, alpha: int):
        R = ref()
        self.seeds = np.ascontiguousarray(seeds, np.uint64)
        W = len(self.seeds)
        tables = np.empty((W, L), np.int32)
        for w, sd in enumerate(self.seeds):
            tables[w] = build_table_fft(random_sequence(int(sd), L))
        self.lut = power_table(L, alpha)
        self.L, self.n, self.W = L, n, W
        self._h = R.ref_walks_create(self.seeds, W, L, n, tables, self.lut)

    def step(self, steps: int = 1):
        """(NSE/s, seconds, per-walk pivot PSL) of `steps` steps of every walk."""
        secs = C.c_double()
        psl = np.zeros(self.W, np.int32)
        rate = ref().ref_walks_step(self._h, steps, C.byref(secs), psl)
        return rate, secs.value, psl

    def close(self):
        if self._h:
            ref().ref_walks_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def fitness(c: np.ndarray, lut: np.ndarray) -> float:
    return lib().orc_fitness(np.ascontiguousarray(c, np.int32), len(c), lut)


def psl(c: np.ndarray) -> int:
    return lib().orc_psl(np.ascontiguousarray(c, np.int32), len(c))


def eval_flip(s, c, j, lut):
    f = C.c_double()
    p = C.c_int32()
    lib().orc_eval_flip(s, c, len(s), j, lut, C.byref(f), C.byref(p))
    return f.value, p.value


def scan(s, c, start, n, lut):
    values = np.zeros(n + 1, np.float64)
    psls = np.zeros(n + 1, np.int32)
    lib().orc_scan(s, c, len(s), start, n, lut, values, psls)
    return values, psls


def reduce(values, psls, n):
    bi, pi = C.c_uint32(), C.c_uint32()
    v = C.c_double()
    pm = C.c_int32()
    rc = lib().orc_reduce(values, psls, n, C.byref(bi), C.byref(v), C.byref(pm), C.byref(pi))
    return rc, bi.value, v.value, pm.value, pi.value


def apply_flip(s, c, j):
    lib().orc_apply_flip(s, c, len(s), j)


def run_search(length, seed, alpha1, alpha2, ls_lmt, flip_lmt, n_lmt, max_nse,
               init=None, events_cap=1 << 16, traces_cap=0):
    p = OrcParams(length, seed, alpha1, alpha2, ls_lmt, flip_lmt, n_lmt, max_nse, None)
    init_arr = None
    if init is not None:
        init_arr = np.ascontiguousarray(init, np.int8)
        p.init = init_arr.ctypes.data
    sol = np.zeros(length, np.int8)
    rec = OrcRecord()
    events = (OrcEvent * max(events_cap, 1))()
    traces = (OrcTrace * max(traces_cap, 1))() if traces_cap else None
    rc = lib().orc_run_search(C.byref(p), sol, C.byref(rec), C.cast(events, C.c_void_p),
                              events_cap, C.cast(traces, C.c_void_p) if traces else None,
                              traces_cap)
    ev = [(events[i].nse, events[i].psl_best, events[i].phase, events[i].kind)
          for i in range(rec.n_events)]
    tr = [(traces[i].nse, traces[i].value_step, traces[i].value_local, traces[i].psl_best,
           traces[i].phase) for i in range(rec.n_traces)] if traces else []
    return rc, rec, sol, ev, tr
