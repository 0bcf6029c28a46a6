"""Wall time of psl_walks_create with seed-only starts (random_sequence on the
device + NTT tables) for 444 m20 walks, repeated (first call pays pool growth)."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_09801_b200 as P  # noqa: E402
L, nw = 1048575, int(os.environ.get("NW", 444))
ctx = P.Context(0)
p = P.SearchParams(length=L, seed=1, alpha1=4, alpha2=P.default_alpha2(L), ls_lmt=2000, flip_lmt=10,
                   n_lmt=1024, stop=P.StopCondition(max_nse=1 + 1024))
for rep in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    w = P.Walks(p, nw, ctx=ctx); torch.cuda.synchronize(); t1 = time.perf_counter()
    w.close()
    print(f"seed-only create of {nw} walks: {1e3 * (t1 - t0):.1f} ms")
