import time, numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2107_09801_b200 as P
ctx = P.Context(0)
L = 1048575
p = P.SearchParams(length=L, seed=1, alpha1=4, alpha2=10, ls_lmt=2000, flip_lmt=10, n_lmt=1024, stop=P.StopCondition(max_nse=1 + 10*1024))
for nw in (296,):
    torch.cuda.synchronize()
    t = time.perf_counter(); w = P.Walks(p, nw, ctx=ctx); torch.cuda.synchronize(); t1 = time.perf_counter()
    print('walks create', nw, t1 - t)
    t = time.perf_counter(); w.step(1); torch.cuda.synchronize(); print('1 step', time.perf_counter() - t)
    t = time.perf_counter(); r = w.records(solutions=True); print('records+solutions', time.perf_counter() - t)
    w.close()
    inits = np.where(np.random.default_rng(1).integers(0, 2, (nw, L)) == 1, -1, 1).astype(np.int8)
    t = time.perf_counter(); w = P.Walks(p, nw, inits=inits, ctx=ctx); torch.cuda.synchronize(); print('create with inits', time.perf_counter() - t)
    w.close()
