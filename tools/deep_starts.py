"""Deep warm starts for the phase-2 golden cases (test infrastructure input).

Runs one long descent per length on the GPU (alpha1 = 4, ls_lmt so large the
walk never restarts, n_lmt 1024) and saves each walk's best sequence as int8
.npy under gpurun_out/.  From such a pivot most 1024-neighbour steps no longer
improve, so the reference's run_search with ls_lmt = 1 switches phase within a
few steps: tests/golden/make_golden.py --phase2 then runs the reference from
these starts (the starts are stored with the fixtures).

  python tools/deep_starts.py  [m16_steps m18_steps m20_steps]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2107_09801_b200 as P  # noqa: E402


def main():
    steps = [int(x) for x in sys.argv[1:4]] or [20000, 6000, 2500]
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    for (m, S) in zip((16, 18, 20), steps):
        if S <= 0:
            continue
        L = (1 << m) - 1
        p = P.SearchParams(length=L, seed=11, alpha1=4, alpha2=P.default_alpha2(L),
                           ls_lmt=1 << 30, flip_lmt=10, n_lmt=1024,
                           stop=P.StopCondition(max_nse=1 + S * 1024))
        t = time.time()
        recs = P.run_walks(p, 2, seeds=[11, 12])
        r = min(recs, key=lambda x: x.psl_best)
        np.save(os.path.join(ROOT, "gpurun_out", f"deep_m{m}.npy"), r.solution_best)
        print(f"m{m}: {S} steps, psl {r.psl_best}, {time.time() - t:.1f} s", flush=True)


if __name__ == "__main__":
    main()
