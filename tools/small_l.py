"""Small-L throughput: K steps of W walks in ONE launch (the bench's shape) vs one
launch per step (tools/step_time.py), certified mode.

    python tools/small_l.py --length 16383 --walks 444 888 1332 --steps 20
"""
import argparse, json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_09801_b200 as P  # noqa: E402


def run(ctx, p, walks, steps, per_launch):
    w = P.Walks(p, walks, ctx=ctx)
    w.step(1)                                   # first step (fitness of the start)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    ctx.set_stream(s.cuda_stream)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    if per_launch:
        for _ in range(steps):
            w.step(1)
    else:
        w.step(steps)
    b.record(s)
    b.synchronize()
    ms = a.elapsed_time(b)
    ctx.set_stream(None)
    w.close()
    return ms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--length", type=int, nargs="+", default=[16383])
    ap.add_argument("--walks", type=int, nargs="+", default=[444])
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    ctx = P.Context(0)
    for L in a.length:
        p = P.default_params(L)
        p.stop = P.StopCondition(max_nse=1 << 62)
        for W in a.walks:
            for per in (False, True):
                ms = run(ctx, p, W, a.steps, per)
                print(json.dumps({"L": L, "walks": W, "steps": a.steps, "launch_per_step": per,
                                  "ms": ms, "us_per_walk_step": 1e3 * ms * 148 / (W * a.steps),
                                  "nse_per_s": W * p.n_lmt * a.steps / (ms * 1e-3)}), flush=True)


if __name__ == "__main__":
    main()
