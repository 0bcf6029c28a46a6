"""ctypes binding of the C ABI in include/pslb200.h (libpslb200.so, built in-tree).

This is the reference-side binding a Python caller uses; the C++ shim in
include/pslb200.hpp is the equivalent for C++ callers.  There is no fallback:
if the shared library is missing, importing the engine raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("PSLB200_LIB") or os.path.join(HERE, "libpslb200.so")  # override: profiling builds

PSL_OK, PSL_ERR_CONFIG, PSL_ERR_OVERFLOW, PSL_ERR_CUDA, PSL_ERR_CAPACITY = 0, 1, 2, 3, 4


class psl_params(C.Structure):
    _fields_ = [("length", C.c_uint32), ("seed", C.c_uint64), ("alpha1", C.c_uint32),
                ("alpha2", C.c_uint32), ("ls_lmt", C.c_uint32), ("flip_lmt", C.c_uint32),
                ("n_lmt", C.c_uint32), ("workers", C.c_uint32), ("has_max_nse", C.c_int32),
                ("max_nse", C.c_uint64), ("has_max_seconds", C.c_int32),
                ("max_seconds", C.c_double), ("init", C.c_void_p)]


class psl_event(C.Structure):
    _fields_ = [("nse", C.c_uint64), ("elapsed_seconds", C.c_double), ("psl_best", C.c_int32),
                ("phase_index", C.c_uint32), ("kind", C.c_uint32)]


class psl_trace(C.Structure):
    _fields_ = [("nse", C.c_uint64), ("value_step", C.c_double), ("value_local", C.c_double),
                ("psl_best", C.c_int32), ("phase_index", C.c_uint32)]


class psl_run_record(C.Structure):
    _fields_ = [("nse", C.c_uint64), ("elapsed_seconds", C.c_double), ("psl_best", C.c_int32),
                ("merit_factor", C.c_double), ("energy", C.c_int64), ("n_events", C.c_uint64),
                ("n_traces", C.c_uint64), ("switches", C.c_uint64)]


psl_event_cb = C.CFUNCTYPE(None, C.POINTER(psl_event), C.c_void_p)
psl_trace_cb = C.CFUNCTYPE(None, C.POINTER(psl_trace), C.c_void_p)


class psl_hooks(C.Structure):
    _fields_ = [("on_event", psl_event_cb), ("on_scan", psl_trace_cb), ("user", C.c_void_p)]


class psl_scan_job(C.Structure):
    _fields_ = [("seq", C.c_void_p), ("table", C.c_void_p), ("length", C.c_uint32),
                ("start", C.c_uint32), ("n", C.c_uint32), ("lut", C.c_void_p),
                ("lut_size", C.c_uint32), ("values", C.c_void_p), ("psls", C.c_void_p)]


class psl_scan_result(C.Structure):
    _fields_ = [("best_index", C.c_uint32), ("value_step", C.c_double),
                ("best_neighbor_psl", C.c_int32), ("best_psl_index", C.c_uint32)]


class psl_walk_record(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("nse", C.c_uint64), ("elapsed_seconds", C.c_double),
                ("psl_best", C.c_int32), ("status", C.c_int32), ("merit_factor", C.c_double),
                ("energy", C.c_int64), ("switches", C.c_uint64), ("steps", C.c_uint64)]


# name -> (restype, argtypes); the full exported surface of include/pslb200.h
SIGNATURES = {
    "psl_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]),
    "psl_ctx_destroy": (None, [C.c_void_p]),
    "psl_ctx_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "psl_ctx_stream": (C.c_void_p, [C.c_void_p]),
    "psl_version": (C.c_char_p, []),
    "psl_kernel_launches": (C.c_uint32, [C.c_void_p]),
    "psl_ctx_set_scan_mode": (C.c_int, [C.c_void_p, C.c_int]),
    "psl_ctx_scan_mode": (C.c_int, [C.c_void_p]),
    "psl_ctx_scan_stats": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                     C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                     C.POINTER(C.c_uint64)]),
    "psl_flip_deltas": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p,
                                  C.c_char_p, C.c_size_t]),
    "psl_fitness": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32,
                              C.c_uint32, C.POINTER(C.c_double), C.c_char_p, C.c_size_t]),
    "psl_ctx_set_cert_check": (C.c_int, [C.c_void_p, C.c_int]),
    "psl_ctx_cert_check_stats": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64),
                                           C.POINTER(C.c_double)]),
    "psl_probe_imma": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.c_char_p, C.c_size_t]),
    "psl_probe_umma": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.c_char_p, C.c_size_t]),
    "psl_probe_peaks": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                  C.POINTER(C.c_double), C.c_char_p, C.c_size_t]),
    "psl_default_alpha2": (C.c_uint32, [C.c_uint32]),
    "psl_default_n_lmt": (C.c_uint32, [C.c_uint32]),
    "psl_default_flip_lmt": (C.c_uint32, [C.c_uint32]),
    "psl_default_params": (None, [C.c_uint32, C.POINTER(psl_params)]),
    "psl_validate_params": (C.c_int, [C.POINTER(psl_params), C.POINTER(psl_params), C.c_char_p,
                                      C.c_size_t, C.c_char_p, C.c_size_t]),
    "psl_pow_int": (C.c_double, [C.c_double, C.c_uint32]),
    "psl_scan": (C.c_int, [C.c_void_p, C.POINTER(psl_scan_job), C.c_char_p, C.c_size_t]),
    "psl_neighborhood_scan": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                        C.c_uint32, C.POINTER(psl_scan_result), C.c_char_p,
                                        C.c_size_t]),
    "psl_evaluate_neighbor": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                        C.POINTER(C.c_double), C.POINTER(C.c_int32), C.c_char_p,
                                        C.c_size_t]),
    "psl_build_table": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p, C.c_char_p,
                                  C.c_size_t]),
    "psl_verify_sequence": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.POINTER(C.c_int32),
                                      C.POINTER(C.c_double), C.POINTER(C.c_int64), C.c_void_p,
                                      C.c_uint32, C.c_char_p, C.c_size_t]),
    "psl_apply_flip": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32,
                                 C.c_char_p, C.c_size_t]),
    "psl_run_search": (C.c_int, [C.c_void_p, C.POINTER(psl_params), C.POINTER(psl_hooks),
                                 C.POINTER(psl_run_record), C.c_void_p, C.c_char_p, C.c_size_t]),
    "psl_walks_create": (C.c_int, [C.c_void_p, C.POINTER(psl_params), C.c_uint32, C.c_void_p,
                                   C.c_void_p, C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]),
    "psl_walks_step": (C.c_int, [C.c_void_p, C.c_uint32, C.c_char_p, C.c_size_t]),
    "psl_walks_run": (C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t]),
    "psl_walks_records": (C.c_int, [C.c_void_p, C.POINTER(psl_walk_record), C.c_void_p,
                                    C.c_char_p, C.c_size_t]),
    "psl_walks_destroy": (None, [C.c_void_p]),
    "psl_run_walks": (C.c_int, [C.c_void_p, C.POINTER(psl_params), C.c_uint32, C.c_void_p,
                                C.c_void_p, C.POINTER(psl_walk_record), C.c_void_p, C.c_char_p,
                                C.c_size_t]),
    "psl_run_walks_multi": (C.c_int, [C.POINTER(C.c_int), C.c_uint32, C.POINTER(psl_params),
                                      C.c_uint32, C.c_void_p, C.c_void_p,
                                      C.POINTER(psl_walk_record), C.c_void_p,
                                      C.POINTER(C.c_uint32), C.POINTER(C.c_double), C.c_char_p,
                                      C.c_size_t]),
}

_lib = None


def lib():
    """Load libpslb200.so; raise loudly if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise RuntimeError(
                f"{SO_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (make -C paper_2107_09801_b200/csrc). There is no CPU fallback.")
        L = C.CDLL(SO_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
