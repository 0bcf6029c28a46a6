"""Run K steps of 148 walks (length argv[2], default m20) in one launch (after one warm step); with the
PSL_PHASE_TIMING build (PSLB200_LIB=build_ablate/lib_pt.so) the kernel prints
per-warp phase cycles of CTA 0 and every CTA's total cycles."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_09801_b200 as P  # noqa: E402
K = int(sys.argv[1]) if len(sys.argv) > 1 else 10
LEN = int(sys.argv[2]) if len(sys.argv) > 2 else 1048575
ctx = P.Context(0)
p = P.default_params(LEN)
p.stop = P.StopCondition(max_nse=1 << 62)
w = P.Walks(p, 148, ctx=ctx)
w.step(1)
torch.cuda.synchronize()
print("=== timed launch", flush=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s = torch.cuda.Stream()
ctx.set_stream(s.cuda_stream)
e0.record(s); w.step(K); e1.record(s); e1.synchronize()
print(f"=== {K} steps {e0.elapsed_time(e1):.2f} ms", flush=True)
