"""Wall-clock breakdown of one e2e psl_run_walks-equivalent call at m20 (148 walks)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_09801_b200 as P  # noqa: E402
L, nw, steps = 1048575, int(os.environ.get("NW", 148)), int(sys.argv[1]) if len(sys.argv) > 1 else 10
ctx = P.Context(0)
p = P.SearchParams(length=L, seed=1, alpha1=4, alpha2=P.default_alpha2(L), ls_lmt=2000, flip_lmt=10,
                   n_lmt=1024, stop=P.StopCondition(max_nse=1 + steps * 1024))
rng = np.random.default_rng(1234)
inits = torch.from_numpy(np.where(rng.integers(0, 2, (nw, L)) == 1, -1, 1).astype(np.int8)).pin_memory().numpy()
seeds = list(range(1, nw + 1))
out = torch.empty((nw, L), dtype=torch.int8).pin_memory().numpy()
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    w = P.Walks(p, nw, seeds=seeds, inits=inits, ctx=ctx); torch.cuda.synchronize(); t1 = time.perf_counter()
    w.step(steps); torch.cuda.synchronize(); t2 = time.perf_counter()
    r = w.records(solutions=True, out=out); torch.cuda.synchronize(); t3 = time.perf_counter()
    w.close(); torch.cuda.synchronize(); t4 = time.perf_counter()
    t5 = time.perf_counter(); rr = P.run_walks(p, nw, seeds=seeds, inits=inits, ctx=ctx, solutions=True, out=out)
    torch.cuda.synchronize(); t6 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms  steps {1e3*(t2-t1):.1f}  records {1e3*(t3-t2):.1f}  close {1e3*(t4-t3):.1f}"
          f"  | run_walks {1e3*(t6-t5):.1f} ms  nse/s {sum(x.nse for x in rr)/(t6-t5)/1e6:.2f} M")
