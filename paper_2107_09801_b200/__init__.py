"""B200-native engine for the two-phase low-PSL binary-sequence search hot path
(arXiv 2107.09801; reference: pslopt).  See DESIGN.md.

The public API mirrors the reference's (pslopt.hpp headers) in
paper_2107_09801_b200.pslopt; compute runs in libpslb200.so (sm_100a kernels
behind the C ABI of include/pslb200.h).
"""
from . import pslopt  # noqa: F401
from .pslopt import (  # noqa: F401
    CapabilityError, ConfigError, Context, ConvergenceEvent, DeviceError, Error, EventKind,
    IoError, NeighborEval, OverflowError, ParseError, PowerTable, RunRecord, ScanResult,
    ScanTrace, SearchHooks, SearchParams, StopCondition, WalkRecord, Walks, apply_flip,
    build_table, default_alpha2, default_context, default_flip_lmt, default_n_lmt, default_params,
    evaluate_neighbor, fitness, flip_deltas, kVersion, merit_factor, neighborhood_scan, pow_int, psl,
    run_search, run_walks, run_walks_multi, scan_values, validate_params, verify_sequence, SequenceReport)

__version__ = kVersion
