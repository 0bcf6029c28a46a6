"""Device time of K search steps (after one warm step) for both scan modes.

    python tools/step_time.py --length 1048575 --walks 296 --steps 5 [--mode auto|exact|both]
"""
import argparse, json, os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_09801_b200 as P  # noqa: E402


def timed(ctx, mode, p, walks, steps):
    ctx.set_scan_mode(mode)
    w = P.Walks(p, walks, ctx=ctx)
    w.step(1)                       # first step: table chain (always exact)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    ctx.set_stream(s.cuda_stream)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    ev[0].record(s)
    for i in range(steps):           # one launch per step: per-step times
        w.step(1)
        ev[i + 1].record(s)
    ev[-1].synchronize()
    per = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
    print("per-step ms:", " ".join(f"{x:.2f}" for x in per), file=sys.stderr)
    ms = sum(per)
    before = ctx.scan_stats()
    w.records()
    after = ctx.scan_stats()
    ctx.set_stream(None)
    w.close()
    return ms, {k: after[k] - before[k] for k in after}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--length", type=int, default=1048575)
    ap.add_argument("--walks", type=int, default=296)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--mode", default="both")
    ap.add_argument("--n-lmt", type=int, default=0)
    a = ap.parse_args()
    ctx = P.Context(0)
    p = P.default_params(a.length)
    if a.n_lmt:
        p.n_lmt = a.n_lmt
    p.stop = P.StopCondition(max_nse=1 << 62)
    out = {"L": a.length, "walks": a.walks, "steps": a.steps, "n_lmt": p.n_lmt}
    for name, mode in (("auto", ctx.SCAN_AUTO), ("exact", ctx.SCAN_EXACT)):
        if a.mode not in ("both", name):
            continue
        ms, st = timed(ctx, mode, p, a.walks, a.steps)
        out[name + "_ms_per_step"] = ms / a.steps
        out[name + "_nse_per_s"] = a.walks * p.n_lmt * a.steps / (ms * 1e-3)
        out[name + "_stats"] = st
    print(json.dumps(out))


if __name__ == "__main__":
    main()
