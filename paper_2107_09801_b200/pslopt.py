"""Host-side mirror of the reference's public API (pslopt, /root/reference/proj).

Same names, argument meaning and error behaviour as the reference headers
(include/pslopt/{search,sequence,errors}.hpp); every compute call goes through
the C ABI in include/pslb200.h into the sm_100a kernels.  Sequences are numpy
int8 arrays of +1/-1, sidelobe tables numpy int32 arrays with table[0] == L.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field, replace
from typing import Callable, Optional, Sequence

import numpy as np

from . import _lib as B

kMinLength = 2                 # sequence.hpp:12
kMaxLength = 1 << 20           # sequence.hpp:13
kVersion = "0.1.0"             # version.hpp:5


# ------------------------------------------------------------------ errors.hpp:8-44

class Error(RuntimeError):
    """Base class for everything this library raises on purpose."""


class ConfigError(Error):
    pass


class OverflowError(Error):  # noqa: A001 -- mirrors pslopt::OverflowError
    pass


class ParseError(Error):
    pass


class IoError(Error):
    pass


class CapabilityError(Error):
    pass


class DeviceError(Error):
    """CUDA device missing or failed (the engine has no CPU fallback)."""


def _raise(rc: int, err: C.Array) -> None:
    msg = err.value.decode(errors="replace")
    if rc == B.PSL_ERR_CONFIG:
        raise ConfigError(msg)
    if rc == B.PSL_ERR_OVERFLOW:
        raise OverflowError(msg)
    raise DeviceError(msg or f"status {rc}")


def _err() -> C.Array:
    return C.create_string_buffer(1024)


# ------------------------------------------------------------------ context

class Context:
    """Owns a device context (psl_ctx); one per GPU per host thread."""

    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        err = _err()
        rc = B.lib().psl_ctx_create(device, C.byref(self._h), err, len(err))
        if rc:
            _raise(rc, err)
        self.device = device

    @property
    def handle(self):
        return self._h

    def set_stream(self, stream_ptr: int | None) -> None:
        B.lib().psl_ctx_set_stream(self._h, C.c_void_p(stream_ptr) if stream_ptr else None)

    def stream(self) -> int:
        return B.lib().psl_ctx_stream(self._h) or 0

    def kernel_launches(self) -> int:
        return B.lib().psl_kernel_launches(self._h)

    SCAN_AUTO, SCAN_EXACT = 0, 1

    def set_scan_mode(self, mode: int) -> None:
        """SCAN_AUTO: certified tensor-core scan where it decides the step,
        exact sweep otherwise (identical results); SCAN_EXACT: exact sweep only."""
        if B.lib().psl_ctx_set_scan_mode(self._h, int(mode)):
            raise ConfigError(f"unknown scan mode {mode}")

    def scan_mode(self) -> int:
        return B.lib().psl_ctx_scan_mode(self._h)

    def scan_stats(self) -> dict:
        """Totals over records read on this context: certified steps, certified
        steps re-scored by the exact sweep, exact value_local chains."""
        a, b, c, d, e = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        B.lib().psl_ctx_scan_stats(self._h, C.byref(a), C.byref(b), C.byref(c), C.byref(d),
                                   C.byref(e))
        return {"certified": a.value, "refined": b.value, "chains": c.value, "mma": d.value,
                "umma": e.value}

    def set_cert_check(self, on: bool) -> None:
        """Certificate check (validation hook): re-score every certified step with
        the exact sweep and test each row's serial double against its interval."""
        B.lib().psl_ctx_set_cert_check(self._h, 1 if on else 0)

    def cert_check_stats(self) -> dict:
        cnt = (C.c_uint64 * 5)()
        mx = (C.c_double * 2)()
        B.lib().psl_ctx_cert_check_stats(self._h, cnt, mx)
        return {"steps": cnt[0], "rows": cnt[1], "violations": cnt[2], "decided": cnt[3],
                "decided_wrong": cnt[4], "tightness": mx[0], "rel_width": mx[1]}

    def probe_umma(self) -> float:
        """tcgen05.mma kind::i8 M128 N64 K32 instructions per second (all SMs)."""
        v = C.c_double()
        err = _err()
        rc = B.lib().psl_probe_umma(self._h, C.byref(v), err, len(err))
        if rc:
            _raise(rc, err)
        return v.value

    def probe_imma(self) -> float:
        """mma.sync m16n8k32 s8 instructions per second on this GPU (all SMs)."""
        v = C.c_double()
        err = _err()
        rc = B.lib().psl_probe_imma(self._h, C.byref(v), err, len(err))
        if rc:
            _raise(rc, err)
        return v.value

    def close(self) -> None:
        if self._h:
            B.lib().psl_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


# ------------------------------------------------------------------ params (search.hpp:21-42)

@dataclass
class StopCondition:
    max_nse: Optional[int] = None
    max_seconds: Optional[float] = None


@dataclass
class SearchParams:
    length: int = 0
    seed: int = 1
    alpha1: int = 4
    alpha2: int = 13
    ls_lmt: int = 2000
    flip_lmt: int = 10
    n_lmt: int = 1024
    workers: int = 1
    stop: StopCondition = field(default_factory=StopCondition)
    init: Optional[np.ndarray] = None

    def __eq__(self, other):
        if not isinstance(other, SearchParams):
            return NotImplemented
        a = replace(self, init=None)
        b = replace(other, init=None)
        if (self.init is None) != (other.init is None):
            return False
        same_init = self.init is None or np.array_equal(self.init, other.init)
        return a.__dict__ == b.__dict__ and same_init


def _to_c(p: SearchParams):
    c = B.psl_params()
    c.length, c.seed = p.length, p.seed
    c.alpha1, c.alpha2, c.ls_lmt, c.flip_lmt = p.alpha1, p.alpha2, p.ls_lmt, p.flip_lmt
    c.n_lmt, c.workers = p.n_lmt, p.workers
    c.has_max_nse = p.stop.max_nse is not None
    c.max_nse = p.stop.max_nse or 0
    c.has_max_seconds = p.stop.max_seconds is not None
    c.max_seconds = float(p.stop.max_seconds or 0.0)
    keep = None
    if p.init is not None:
        keep = np.ascontiguousarray(p.init, np.int8).reshape(-1)
        if keep.size != p.length:
            # the C ABI reads `length` elements: report the checks that precede
            # this one first (search.cpp:40-71), then the reference's message (:72-76)
            err = _err()
            rc = B.lib().psl_validate_params(C.byref(c), None, None, 0, err, len(err))
            if rc:
                _raise(rc, err)
            raise ConfigError(f"warm-start sequence has length {keep.size}, expected {p.length}")
        c.init = keep.ctypes.data
    return c, keep


def default_alpha2(length: int) -> int:            # search.cpp:19-23
    return B.lib().psl_default_alpha2(length)


def default_n_lmt(length: int) -> int:             # search.cpp:25
    return B.lib().psl_default_n_lmt(length)


def default_flip_lmt(length: int) -> int:          # search.cpp:27
    return B.lib().psl_default_flip_lmt(length)


def default_params(length: int) -> SearchParams:   # search.cpp:29-38
    return SearchParams(length=length, alpha1=4, alpha2=default_alpha2(length), ls_lmt=2000,
                        flip_lmt=default_flip_lmt(length), n_lmt=default_n_lmt(length))


def validate_params(params: SearchParams, warning: Optional[list] = None) -> SearchParams:
    """search.cpp:40-94: raises ConfigError; clamps n_lmt / flip_lmt."""
    c, keep = _to_c(params)
    out = B.psl_params()
    warn, err = C.create_string_buffer(1024), _err()
    rc = B.lib().psl_validate_params(C.byref(c), C.byref(out), warn, len(warn), err, len(err))
    if rc:
        _raise(rc, err)
    if warning is not None and warn.value:
        warning.append(warn.value.decode())
    return replace(params, n_lmt=out.n_lmt, flip_lmt=out.flip_lmt,
                   init=None if params.init is None else np.array(params.init, np.int8),
                   stop=StopCondition(params.stop.max_nse, params.stop.max_seconds))


# ------------------------------------------------------------------ observability (search.hpp:74-103)

class EventKind(enum.IntEnum):
    kImprovedPsl = 0
    kPhaseSwitch = 1
    kLocalBestImproved = 2


_KIND_NAMES = {EventKind.kImprovedPsl: "improved-psl", EventKind.kPhaseSwitch: "phase-switch",
               EventKind.kLocalBestImproved: "local-best-improved"}


def to_string(kind: EventKind) -> str:              # search.cpp:100-107
    return _KIND_NAMES.get(EventKind(kind), "unknown")


def event_kind_from_string(name: str) -> EventKind:  # search.cpp:109-114
    for k, v in _KIND_NAMES.items():
        if v == name:
            return k
    raise ParseError(f"unknown event kind '{name}'")


@dataclass
class ConvergenceEvent:
    nse: int
    elapsed_seconds: float
    psl_best: int
    phase_index: int
    kind: EventKind


@dataclass
class ScanTrace:
    nse: int
    value_step: float
    value_local: float
    psl_best: int
    phase_index: int


@dataclass
class SearchHooks:
    on_event: Optional[Callable[[ConvergenceEvent], None]] = None
    on_scan: Optional[Callable[[ScanTrace], None]] = None


@dataclass
class RunRecord:                                     # search.hpp:109-120
    params: SearchParams
    solution_best: np.ndarray
    psl_best: int
    merit_factor: float
    nse: int
    elapsed_seconds: float
    events: list
    solver_version: str


@dataclass
class ScanResult:                                    # search.hpp:136-141
    best_index: int
    value_step: float
    best_neighbor_psl: int
    best_psl_index: int


@dataclass
class NeighborEval:                                  # sequence.hpp:102-105
    fitness: float
    psl: int


# ------------------------------------------------------------------ sequence core

def _seq(s) -> np.ndarray:
    a = np.ascontiguousarray(s, dtype=np.int8)
    if a.ndim != 1:
        raise ConfigError("sequence must be one-dimensional")
    return a


def pow_int(base: float, exp: int) -> float:        # sequence.cpp:95-105
    return B.lib().psl_pow_int(float(base), exp)


class PowerTable:                                    # sequence.hpp:72-84
    def __init__(self, max_abs_value: int, alpha: int):
        if alpha < 1:
            raise ConfigError("fitness exponent must be >= 1")
        self.alpha = alpha
        self.lut = np.array([pow_int(float(a), alpha) for a in range(max_abs_value + 1)],
                            np.float64) if max_abs_value < 4096 else _fast_lut(max_abs_value, alpha)

    def __getitem__(self, a):
        return self.lut[a]

    def size(self) -> int:
        return len(self.lut)


def _fast_lut(max_abs: int, alpha: int) -> np.ndarray:
    # identical to pow_int: binary exponentiation, lowest bit first, RN multiplies
    base = np.arange(max_abs + 1, dtype=np.float64)
    result = np.ones_like(base)
    factor = base.copy()
    e = alpha
    while e:
        if e & 1:
            result = result * factor
        e >>= 1
        if e:
            factor = factor * factor
    return result


def build_table(seq, ctx: Context | None = None) -> np.ndarray:
    """SidelobeTable::build (sequence.cpp:46-60) on the device."""
    s = _seq(seq)
    ctx = ctx or default_context()
    out = np.empty(len(s), np.int32)
    err = _err()
    rc = B.lib().psl_build_table(ctx.handle, s.ctypes.data, len(s), out.ctypes.data, err, len(err))
    if rc:
        _raise(rc, err)
    return out


def psl(table) -> int:                               # sequence.cpp:84-93
    t = np.asarray(table)
    return int(np.abs(t[1:]).max()) if len(t) > 1 else 0


def merit_factor(table) -> float:                    # sequence.cpp:143-152
    t = np.asarray(table, np.int64)
    energy = int((t[1:] * t[1:]).sum())
    L = len(t)
    return (float(L) * float(L)) / (2.0 * float(energy))


def fitness(table, pow_or_alpha, ctx: Context | None = None) -> float:   # sequence.cpp:117-141
    """The serial ascending-k double sum of |C_k|^alpha, on the device
    (psl_fitness); OverflowError when it leaves the finite range."""
    t = np.ascontiguousarray(table, np.int32)
    lut, alpha = _lut_for(len(t), pow_or_alpha)
    lut = np.ascontiguousarray(lut, np.float64)
    ctx = ctx or default_context()
    v = C.c_double()
    err = _err()
    rc = B.lib().psl_fitness(ctx.handle, t.ctypes.data, len(t), lut.ctypes.data, len(lut), alpha,
                             C.byref(v), err, len(err))
    if rc:
        _raise(rc, err)
    return v.value


def flip_deltas(seq, j: int, ctx: Context | None = None) -> np.ndarray:   # sequence.cpp:154-172
    """delta_k of flipping position j (out[0] = 0), on the device."""
    s = _seq(seq)
    out = np.zeros(len(s), np.int32)
    ctx = ctx or default_context()
    err = _err()
    rc = B.lib().psl_flip_deltas(ctx.handle, s.ctypes.data, len(s), j, out.ctypes.data, err,
                                 len(err))
    if rc:
        _raise(rc, err)
    return out


@dataclass
class SequenceReport:                                # oracle.hpp SequenceReport
    length: int
    psl: int
    merit_factor: float
    sidelobe_histogram: np.ndarray


def verify_sequence(seq, ctx: Context | None = None) -> SequenceReport:
    """oracle::verify_sequence (oracle.cpp:172-197) on the device."""
    s = _seq(seq)
    ctx = ctx or default_context()
    L = len(s)
    psl_, mf, en = C.c_int32(), C.c_double(), C.c_int64()
    hist = np.zeros(L + 1, np.uint64)
    err = _err()
    rc = B.lib().psl_verify_sequence(ctx.handle, s.ctypes.data, L, C.byref(psl_), C.byref(mf),
                                     C.byref(en), hist.ctypes.data, L + 1, err, len(err))
    if rc:
        _raise(rc, err)
    return SequenceReport(L, psl_.value, mf.value, hist[:psl_.value + 1].copy())


def apply_flip(seq: np.ndarray, table: np.ndarray, j: int, ctx: Context | None = None) -> None:
    """apply_flip (sequence.cpp:198-224), in place, on the device."""
    if seq.dtype != np.int8 or table.dtype != np.int32 or not seq.flags.c_contiguous:
        raise ConfigError("apply_flip needs contiguous int8 sequence and int32 table")
    ctx = ctx or default_context()
    err = _err()
    rc = B.lib().psl_apply_flip(ctx.handle, seq.ctypes.data, table.ctypes.data, len(seq), j,
                                err, len(err))
    if rc:
        _raise(rc, err)


def _lut_for(L: int, pow_or_alpha):
    if isinstance(pow_or_alpha, PowerTable):
        return pow_or_alpha.lut, pow_or_alpha.alpha
    return PowerTable(L, int(pow_or_alpha)).lut, int(pow_or_alpha)


def evaluate_neighbor(seq, table, j: int, pow_or_alpha, ctx: Context | None = None) -> NeighborEval:
    """evaluate_neighbor (sequence.cpp:174-196)."""
    s = _seq(seq)
    t = np.ascontiguousarray(table, np.int32)
    if len(t) != len(s):
        raise ConfigError("sidelobe table length does not match sequence length")
    lut, alpha = _lut_for(len(s), pow_or_alpha)
    lut = np.ascontiguousarray(lut, np.float64)
    ctx = ctx or default_context()
    f, p = C.c_double(), C.c_int32()
    err = _err()
    rc = B.lib().psl_evaluate_neighbor(ctx.handle, s.ctypes.data, t.ctypes.data, lut.ctypes.data,
                                       len(lut), alpha, len(s), j, C.byref(f), C.byref(p), err,
                                       len(err))
    if rc:
        _raise(rc, err)
    return NeighborEval(f.value, p.value)


def scan_values(seq, table, start: int, n: int, lut, ctx: Context | None = None):
    """The ScanJob operator seam (search.cpp:156-175): values/psls slots 1..n."""
    s = _seq(seq)
    t = np.ascontiguousarray(table, np.int32)
    lut = np.ascontiguousarray(lut, np.float64)
    values = np.zeros(n + 1, np.float64)
    psls = np.zeros(n + 1, np.int32)
    job = B.psl_scan_job(s.ctypes.data, t.ctypes.data, len(s), start, n, lut.ctypes.data,
                         len(lut), values.ctypes.data, psls.ctypes.data)
    ctx = ctx or default_context()
    err = _err()
    rc = B.lib().psl_scan(ctx.handle, C.byref(job), err, len(err))
    if rc:
        _raise(rc, err)
    return values, psls


def neighborhood_scan(pivot, table, pow: PowerTable, start: int, n: int,
                      ctx: Context | None = None) -> ScanResult:
    """neighborhood_scan (search.cpp:296-321)."""
    s = _seq(pivot)
    t = np.ascontiguousarray(table, np.int32)
    if len(t) != len(s):
        raise ConfigError("sidelobe table length does not match sequence length")
    lut = np.ascontiguousarray(pow.lut, np.float64)
    ctx = ctx or default_context()
    out = B.psl_scan_result()
    err = _err()
    rc = B.lib().psl_neighborhood_scan(ctx.handle, s.ctypes.data, t.ctypes.data, lut.ctypes.data,
                                       len(lut), pow.alpha, len(s), start, n, C.byref(out), err,
                                       len(err))
    if rc:
        _raise(rc, err)
    return ScanResult(out.best_index, out.value_step, out.best_neighbor_psl, out.best_psl_index)


# ------------------------------------------------------------------ run_search (search.cpp:327-430)

def run_search(params: SearchParams, hooks: SearchHooks | None = None,
               ctx: Context | None = None) -> RunRecord:
    p = validate_params(params)
    c, keep = _to_c(p)
    ctx = ctx or default_context()
    events: list[ConvergenceEvent] = []
    hooks = hooks or SearchHooks()

    def _on_event(ptr, _user):
        e = ptr.contents
        ev = ConvergenceEvent(e.nse, e.elapsed_seconds, e.psl_best, e.phase_index,
                              EventKind(e.kind))
        events.append(ev)
        if hooks.on_event:
            hooks.on_event(ev)

    def _on_scan(ptr, _user):
        t = ptr.contents
        hooks.on_scan(ScanTrace(t.nse, t.value_step, t.value_local, t.psl_best, t.phase_index))

    cb_e = B.psl_event_cb(_on_event)
    cb_s = B.psl_trace_cb(_on_scan) if hooks.on_scan else B.psl_trace_cb()
    h = B.psl_hooks(cb_e, cb_s, None)
    rec = B.psl_run_record()
    sol = np.zeros(p.length, np.int8)
    err = _err()
    rc = B.lib().psl_run_search(ctx.handle, C.byref(c), C.byref(h), C.byref(rec),
                                sol.ctypes.data, err, len(err))
    del keep
    if rc:
        _raise(rc, err)
    return RunRecord(p, sol, rec.psl_best, rec.merit_factor, rec.nse, rec.elapsed_seconds,
                     events, kVersion)


# ------------------------------------------------------------------ many walks

@dataclass
class WalkRecord:
    seed: int
    nse: int
    elapsed_seconds: float
    psl_best: int
    status: int
    merit_factor: float
    energy: int
    switches: int
    steps: int
    solution_best: Optional[np.ndarray] = None


def _walk_inputs(p: SearchParams, n_walks: int, seeds, inits):
    """seeds / warm starts for n_walks walks, checked before the C ABI reads
    8 n_walks seed bytes and n_walks x L start bytes (one (L,) start is given
    to every walk)."""
    if n_walks < 1:
        raise ConfigError("n_walks must be >= 1")
    seeds_arr = None
    if seeds is not None:
        seeds_arr = np.ascontiguousarray(seeds, np.uint64).reshape(-1)
        if seeds_arr.size != n_walks:
            raise ConfigError(f"{seeds_arr.size} seeds given for {n_walks} walks")
    inits_arr = None
    if inits is not None:
        inits_arr = np.asarray(inits)
        if inits_arr.shape == (p.length,):
            inits_arr = np.broadcast_to(inits_arr, (n_walks, p.length))
        if inits_arr.shape != (n_walks, p.length):
            raise ConfigError(f"warm starts have shape {tuple(np.shape(inits))}, expected "
                              f"({n_walks}, {p.length}) or ({p.length},)")
        inits_arr = np.ascontiguousarray(inits_arr, np.int8)
    return seeds_arr, inits_arr


class Walks:
    """n independent walks (one CTA each) advanced on the device in lock-step
    batches of steps; walk w uses seed params.seed + w unless seeds is given."""

    def __init__(self, params: SearchParams, n_walks: int, seeds: Sequence[int] | None = None,
                 inits: np.ndarray | None = None, ctx: Context | None = None):
        p = validate_params(params)
        self.params = p
        self.n_walks = n_walks
        self._h = C.c_void_p()
        seeds_arr, inits_arr = _walk_inputs(p, n_walks, seeds, inits)
        self.ctx = ctx or default_context()
        c, keep = _to_c(p)
        self._h = C.c_void_p()
        err = _err()
        rc = B.lib().psl_walks_create(self.ctx.handle, C.byref(c), n_walks,
                                      seeds_arr.ctypes.data if seeds_arr is not None else None,
                                      inits_arr.ctypes.data if inits_arr is not None else None,
                                      C.byref(self._h), err, len(err))
        del keep
        if rc:
            _raise(rc, err)

    def step(self, steps: int) -> None:
        err = _err()
        rc = B.lib().psl_walks_step(self._h, steps, err, len(err))
        if rc:
            _raise(rc, err)

    def run(self) -> None:
        err = _err()
        rc = B.lib().psl_walks_run(self._h, err, len(err))
        if rc:
            _raise(rc, err)

    def records(self, solutions: bool = False, out: np.ndarray | None = None) -> list[WalkRecord]:
        """Per-walk records; with solutions=True also each walk's best sequence
        (int8 +-1), written into `out` (n_walks x L int8, C-contiguous; e.g. a
        pinned buffer the caller reuses) when given."""
        recs = (B.psl_walk_record * self.n_walks)()
        sol = None
        if solutions:
            if out is not None:
                if (out.dtype != np.int8 or out.shape != (self.n_walks, self.params.length)
                        or not out.flags.c_contiguous):
                    raise ValueError("out must be a C-contiguous int8 array of shape (n_walks, length)")
                sol = out
            else:
                sol = np.zeros((self.n_walks, self.params.length), np.int8)
        err = _err()
        rc = B.lib().psl_walks_records(self._h, recs, sol.ctypes.data if sol is not None else None,
                                       err, len(err))
        if rc:
            _raise(rc, err)
        return [WalkRecord(r.seed, r.nse, r.elapsed_seconds, r.psl_best, r.status, r.merit_factor,
                           r.energy, r.switches, r.steps, None if sol is None else sol[i])
                for i, r in enumerate(recs)]

    def close(self) -> None:
        if self._h:
            B.lib().psl_walks_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_walks(params: SearchParams, n_walks: int, seeds=None, inits=None,
              ctx: Context | None = None, solutions: bool = True,
              out: np.ndarray | None = None) -> list[WalkRecord]:
    """One psl_run_walks call: create, run every walk to its stop, records.
    With a pinned `out` buffer each walk's kernel writes its best sequence
    straight into it when the walk stops (the D2H overlaps later walks)."""
    p = validate_params(params)
    seeds_arr, inits_arr = _walk_inputs(p, n_walks, seeds, inits)
    ctx = ctx or default_context()
    c, keep = _to_c(p)
    recs = (B.psl_walk_record * n_walks)()
    sol = None
    if solutions:
        if out is not None:
            if out.dtype != np.int8 or out.shape != (n_walks, p.length) or not out.flags.c_contiguous:
                raise ValueError("out must be a C-contiguous int8 array of shape (n_walks, length)")
            sol = out
        else:
            sol = np.zeros((n_walks, p.length), np.int8)
    err = _err()
    rc = B.lib().psl_run_walks(ctx.handle, C.byref(c), n_walks,
                               seeds_arr.ctypes.data if seeds_arr is not None else None,
                               inits_arr.ctypes.data if inits_arr is not None else None,
                               recs, sol.ctypes.data if sol is not None else None, err, len(err))
    del keep
    if rc:
        _raise(rc, err)
    return [WalkRecord(r.seed, r.nse, r.elapsed_seconds, r.psl_best, r.status, r.merit_factor,
                       r.energy, r.switches, r.steps, None if sol is None else sol[i])
            for i, r in enumerate(recs)]


def run_walks_multi(params: SearchParams, n_walks: int, devices: Sequence[int], seeds=None,
                    inits=None, solutions: bool = True):
    """psl_run_walks_multi: walks split into contiguous blocks over `devices`
    (one host thread + context per device, no per-step communication), records
    gathered on the host in global walk order.  Returns (records, best_walk,
    per-device seconds); best_walk minimises (psl_best, walk index)."""
    p = validate_params(params)
    seeds_arr, inits_arr = _walk_inputs(p, n_walks, seeds, inits)
    devs = (C.c_int * len(devices))(*devices)
    c, keep = _to_c(p)
    recs = (B.psl_walk_record * n_walks)()
    sol = np.zeros((n_walks, p.length), np.int8) if solutions else None
    best = C.c_uint32()
    secs = (C.c_double * len(devices))()
    err = _err()
    rc = B.lib().psl_run_walks_multi(devs, len(devices), C.byref(c), n_walks,
                                     seeds_arr.ctypes.data if seeds_arr is not None else None,
                                     inits_arr.ctypes.data if inits_arr is not None else None,
                                     recs, sol.ctypes.data if sol is not None else None,
                                     C.byref(best), secs, err, len(err))
    del keep
    if rc:
        _raise(rc, err)
    out = [WalkRecord(r.seed, r.nse, r.elapsed_seconds, r.psl_best, r.status, r.merit_factor,
                      r.energy, r.switches, r.steps, None if sol is None else sol[i])
           for i, r in enumerate(recs)]
    return out, best.value, list(secs)
