"""Long fixed-wall-time run of W independent two-phase walks (reference defaults),
logging the best PSL as it evolves: one JSON line per launch of `--chunk` steps.
Saves the best sequence (int8 +-1, .npy) at the end, re-verified from a fresh table.

    python tools/long_run.py --m 20 --seconds 7200 --out gpurun_out/long_m20
"""
import argparse, json, math, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_09801_b200 as P  # noqa: E402

PAPER_BEST = {14: 101, 15: 146, 16: 209, 17: 301, 18: 434, 19: 628, 20: 901}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=20)
    ap.add_argument("--seconds", type=float, default=600.0)
    ap.add_argument("--walks", type=int, default=148)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--chunk", type=int, default=10000, help="steps per launch between log lines")
    ap.add_argument("--out", default="gpurun_out/long_run")
    a = ap.parse_args()
    L = (1 << a.m) - 1
    ctx = P.Context(0)
    p = P.default_params(L)
    p.seed = a.seed
    p.stop = P.StopCondition(max_seconds=a.seconds)
    w = P.Walks(p, a.walks, ctx=ctx)
    t0 = time.perf_counter()
    log = open(a.out + ".jsonl", "w")
    while True:
        w.step(a.chunk)
        recs = w.records()
        psls = np.array([r.psl_best for r in recs])
        line = {"m": a.m, "L": L, "walks": a.walks, "wall_seconds": time.perf_counter() - t0,
                "best_psl": int(psls.min()), "mean_psl": float(psls.mean()),
                "best_psl_over_sqrtL": float(psls.min() / math.sqrt(L)),
                "walks_switched": int(sum(1 for r in recs if r.switches > 0)),
                "switches_total": int(sum(r.switches for r in recs)),
                "steps_mean": float(np.mean([r.steps for r in recs])),
                "nse_total": int(sum(r.nse for r in recs)),
                "walk_seconds_min": float(min(r.elapsed_seconds for r in recs)),
                "paper_best_4day_a100": PAPER_BEST.get(a.m)}
        print(json.dumps(line), flush=True)
        log.write(json.dumps(line) + "\n"); log.flush()
        if line["walk_seconds_min"] >= a.seconds or line["wall_seconds"] >= a.seconds + 60:
            break
    recs = w.records(solutions=True)
    best = min(range(len(recs)), key=lambda i: recs[i].psl_best)
    sol = recs[best].solution_best
    t = P.build_table(sol, ctx)
    assert P.psl(t) == recs[best].psl_best
    np.save(a.out + "_best.npy", sol.astype(np.int8))
    fin = {"final": True, "best_psl": int(recs[best].psl_best), "best_walk_seed": int(recs[best].seed),
           "merit_factor": recs[best].merit_factor, "verified": True}
    print(json.dumps(fin), flush=True)
    log.write(json.dumps(fin) + "\n")
    w.close()


if __name__ == "__main__":
    main()
