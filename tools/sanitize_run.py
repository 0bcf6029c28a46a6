"""Small engine runs for compute-sanitizer (memcheck / racecheck / synccheck).

  compute-sanitizer --tool racecheck python tools/sanitize_run.py [L] [mode]

mode: auto (certified tensor-core scan, the default path) or exact (serial-chain
sweep).  ls_lmt = 2 forces phase switches and restarts inside the few steps, so
the restart (flip_lmt random flips, snapshot restore, chain fitness) paths run.
The records are checked against the CPU oracle (test infrastructure only)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2107_09801_b200 as P  # noqa: E402
from oracle import oracle_py as O  # noqa: E402


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    mode = sys.argv[2] if len(sys.argv) > 2 else "auto"
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    ctx = P.default_context()
    ctx.set_scan_mode(ctx.SCAN_EXACT if mode == "exact" else ctx.SCAN_AUTO)
    n = min(L, 1024)
    p = P.SearchParams(length=L, seed=3, alpha1=4, alpha2=P.default_alpha2(L), ls_lmt=2,
                       flip_lmt=min(L, 10), n_lmt=n,
                       stop=P.StopCondition(max_nse=1 + steps * n))
    r = P.run_search(p)
    rc, o, osol, oev, _ = O.run_search(L, 3, 4, P.default_alpha2(L), 2, min(L, 10), n,
                                       1 + steps * n, traces_cap=0)
    assert rc == 0
    assert (r.nse, r.psl_best) == (o.nse, o.psl_best), ((r.nse, r.psl_best), (o.nse, o.psl_best))
    assert np.array_equal(r.solution_best, osol)
    assert [(e.nse, e.psl_best, e.phase_index, int(e.kind)) for e in r.events] == oev
    switches = sum(1 for e in r.events if int(e.kind) == int(P.EventKind.kPhaseSwitch))
    # several walks in one launch (the bench's many-walk path)
    w = P.Walks(p, 3, seeds=[3, 4, 5], ctx=ctx)
    w.run()
    recs = w.records(solutions=True)
    w.close()
    assert recs[0].psl_best == r.psl_best and np.array_equal(recs[0].solution_best, osol)
    print(f"sanitize_run ok: L={L} mode={mode} nse={r.nse} psl={r.psl_best} "
          f"switches={switches} stats={ctx.scan_stats()}")


if __name__ == "__main__":
    main()
