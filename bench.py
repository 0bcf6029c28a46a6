#!/usr/bin/env python
"""Benchmark: flip-evaluations/s (NSE/s) of the two-phase low-PSL search at
L = 2^20 - 1 (BASELINE.json metric), one JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step = one search step of every walk on every GPU: each walk scans its
n_lmt = 1024 one-flip neighbours (1024 x (L-1) flip x shift cells), reduces,
moves (and restarts when the phase rule fires), all on the device.  Walks are
independent (seed = seed0 + global walk id), one CTA per SM at a time, so
per-GPU work is fixed as N grows ("scaling": "weak").  Inputs are synthetic
random start sequences (random_sequence(L, Rng(seed))), the reference's own.

--gpus N > 1 runs one process per GPU: under torchrun (WORLD_SIZE set) the
ranks are the launcher's; started directly, bench.py re-launches itself under
torch.distributed.run with N processes.  World size must equal N.

--impl reference times the reference's CPU implementation of the same path
(oracle/_ref/libpslref.so, compiled from the unmodified reference sources) on
all host cores: one independent walk per host thread (walk w = run_search
(seed w)'s pivot), each step = the reference's run_search step (start draw,
n_lmt detail::eval_flip scores, first-minimum argmin, apply_flip).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L_DEFAULT = (1 << 20) - 1
A100_M20_NSE = 85062.0   # BASELINE.md / PAPER.md:342-359, A100, L = 1048575 (N_lmt = 6912)
METRIC = "flip-evals/sec (NSE/s) at L=2^20-1"
INT_OPS_PER_CELL = 4     # delta, +c, abs, max per flip x shift cell


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40,
                    help="timed search steps, all in one launch like psl_walks_run (long launches amortise the end-of-launch tail of the walk CTAs)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--length", type=int, default=L_DEFAULT)
    ap.add_argument("--walks", type=int, default=0,
                    help="walks per GPU (0 = three per SM: the hardware runs them as three waves "
                         "of one 512-thread walk CTA per SM, which evens out per-walk work)")
    ap.add_argument("--n-lmt", type=int, default=1024)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--e2e-steps", type=int, default=10, help="search steps per e2e call")
    ap.add_argument("--e2e-reps", type=int, default=2, help="timed e2e calls")
    ap.add_argument("--exact-steps", type=int, default=3,
                    help="timed steps of the exact (value-exact) sweep sub-measurement (0 = skip)")
    ap.add_argument("--cpu-steps", type=int, default=2, help="steps of the cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-probes", action="store_true", help="skip the live peak probes")
    return ap.parse_args()


# ---------------------------------------------------------------- launch

def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch_under_torchrun(n: int) -> int:
    """One process per GPU: re-run this script under torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, cwd=ROOT)


# ---------------------------------------------------------------- clocks

class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        # NVML at 10 ms (a timed region of K steps lasts ~0.1-0.3 s); nvidia-smi otherwise
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.device)
            mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            bits = (0x8, 0x40, 0x20, 0x4)   # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
            while not self._stop.is_set():
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                rs = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append([str(sm), str(mx), hex(rs)] +
                                 ["Active" if rs & b else "Not Active" for b in bits])
                self._stop.wait(0.01)
            return
        except Exception:
            pass
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True,
                    timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------- CPU reference

def host_info() -> dict:
    info = {"threads": os.cpu_count() or 1, "model": None, "threads_per_core": None}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            if k.strip() == "Model name":
                info["model"] = v.strip()
            elif k.strip() == "Thread(s) per core":
                info["threads_per_core"] = int(v.strip())
    except Exception:
        pass
    info["smt"] = None if info["threads_per_core"] is None else info["threads_per_core"] > 1
    return info


def reference_walks(L: int, n: int, seed0: int):
    """One reference walk per host thread (oracle/_ref, unmodified reference
    code): walk w = run_search(seed0 + w)'s pivot and RNG; setup untimed."""
    from oracle import oracle_py as O
    threads = os.cpu_count() or 1
    return O.RefWalks([seed0 + w for w in range(threads)], L, n, 4), threads


def sample_desc(threads: int, L: int, n: int, steps: int, info: dict) -> str:
    return (f"{threads} host threads, one independent walk each (walk w = run_search(seed w)'s "
            f"pivot, L={L}, alpha1=4), {steps} step(s) of the reference's run_search loop body "
            f"per walk: rng.bounded(L) start, {n} detail::eval_flip (sequence.hpp:126-162) "
            f"scores, first-minimum argmin, apply_flip; pivot tables built untimed "
            f"(FFT, pinned to SidelobeTable::build); host {info.get('model')}, "
            f"SMT {'on' if info.get('smt') else 'off' if info.get('smt') is not None else '?'}")


def run_reference_arm(args, rank: int):
    if rank != 0:
        return
    from oracle import oracle_py as O
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libpslref.so not built (needs /root/reference at build time)"}))
        return
    L, n = args.length, args.n_lmt
    info = host_info()
    W, threads = reference_walks(L, n, args.seed)
    for _ in range(args.warmup):
        W.step(1)
    total = 0.0
    for _ in range(args.steps):
        _, secs, _ = W.step(1)
        total += secs
    W.close()
    nse = float(threads) * n * args.steps
    value = nse / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "NSE/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": value / A100_M20_NSE, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"m20: L={L}, {threads} walks (one per host thread), n_lmt={n}",
                   "L": L, "n_lmt": n, "host_threads": threads, "host": info,
                   "step": "every host thread advances its own walk by one run_search step"},
        "cpu_baseline": {"value": value, "unit": "NSE/s", "cores": threads, "kind": "reference",
                         "sample": sample_desc(threads, L, n, args.steps, info)},
        "e2e": {"value": value, "unit": "NSE/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "cells_per_s": value * (L - 1),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- ours

def measured_peaks() -> dict:
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def records_sha(rows) -> str:
    h = hashlib.sha256()
    for r in rows:
        h.update(json.dumps(r).encode())
    return h.hexdigest()


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args.gpus))
    if world != args.gpus:
        print(f"bench.py: world size {world} != --gpus {args.gpus}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference_arm(args, rank)
        return

    import torch
    import torch.distributed as dist

    import paper_2107_09801_b200 as P
    from paper_2107_09801_b200 import dist as D

    # one GPU per rank; PSLB200_BENCH_SAME_DEVICE=1 puts every rank on GPU 0
    # (the 2-process test of this path on a 1-GPU box, with gloo)
    device = 0 if os.environ.get("PSLB200_BENCH_SAME_DEVICE") == "1" else local_rank
    backend = os.environ.get("PSLB200_BENCH_BACKEND", "nccl")
    torch.cuda.set_device(device)
    dev = torch.device("cuda", device)
    cdev = dev if backend == "nccl" else torch.device("cpu")   # collective tensors
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    ctx = P.Context(device)
    # a dedicated (non-default) stream shared by the engine and the CUDA events
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    nsm = torch.cuda.get_device_properties(device).multi_processor_count
    # one 512-thread walk CTA per SM at a time (~211 KB smem); three waves of
    # walks per launch: a CTA that finishes its K steps early hands its SM to the
    # next walk (measured: 148 walks 24.0, 296 25.1, 444 25.6 M NSE/s)
    n_walks = args.walks or 3 * nsm
    L, n = args.length, args.n_lmt
    total_steps = args.warmup + args.steps + 4

    def params(steps_budget):
        return P.SearchParams(length=L, seed=args.seed, alpha1=4, alpha2=P.default_alpha2(L),
                              ls_lmt=2000, flip_lmt=min(L, 10), n_lmt=n,
                              stop=P.StopCondition(max_nse=1 + steps_budget * (n + 1)))

    # rank r runs global walks r*W .. r*W + W - 1 (seed = seed0 + global id)
    seeds = [args.seed + rank * n_walks + w for w in range(n_walks)]

    # roofline denominators measured on this GPU, now
    import ctypes
    dadd, lds, mhz = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    umma_per_s = mma_per_s = None
    if not args.no_probes:
        err = ctypes.create_string_buffer(256)
        P._lib.lib().psl_probe_peaks(ctx.handle, ctypes.byref(dadd), ctypes.byref(lds),
                                     ctypes.byref(mhz), err, 256)
        mma_per_s = ctx.probe_imma()
        umma_per_s = ctx.probe_umma()

    # setup: pivots (random_sequence), tables (NTT) -- untimed, like the reference
    t_setup = time.perf_counter()
    walks = P.Walks(params(total_steps), n_walks, seeds=seeds, ctx=ctx)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup

    for _ in range(args.warmup):
        walks.step(1)
    torch.cuda.synchronize()
    r0 = walks.records()
    nse0 = sum(r.nse for r in r0)
    stats0 = ctx.scan_stats()
    launches0 = ctx.kernel_launches()
    e_start = torch.cuda.Event(enable_timing=True)
    e_end = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(device) as clocks:
        e_start.record(stream)
        # one persistent launch advances every walk by exactly K steps (walks
        # progress independently inside it; no per-step host round trip)
        walks.step(args.steps)
        e_end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e_start.elapsed_time(e_end)
    launches = ctx.kernel_launches() - launches0
    r1 = walks.records(solutions=True)
    stats1 = ctx.scan_stats()
    scan = {k: stats1[k] - stats0[k] for k in stats1}
    nse_local = sum(r.nse for r in r1) - nse0
    max_ms = D.max_over_ranks(ms, cdev)
    nse_total = D.sum_over_ranks(float(nse_local), cdev)
    value = nse_total / (max_ms * 1e-3)
    # end-of-run best-PSL reduction across GPUs (outside the timed region)
    best_psl, best_walk, _ = D.reduce_best([r.psl_best for r in r1], seeds,
                                           [r.solution_best for r in r1], L, device=cdev)
    mine = [[int(s), int(r.nse), int(r.psl_best), int(r.energy), int(r.switches), int(r.steps)]
            for s, r in zip(seeds, r1)]
    if world > 1:
        allrows = [None] * world
        dist.all_gather_object(allrows, mine)
        rows = [x for part in allrows for x in part]
    else:
        rows = mine
    walks.close()

    # dominant kernel: run_kernel, one launch for the K timed steps.  Steps are
    # scored by the certified scan: the correlation on tcgen05
    # (kind::i8 M128 N64 K32, accumulators in TMEM), the zone-1 cross term on
    # mma.sync m16n8k32, the exact DADD sweep only where intervals cannot decide.
    # achieved = int8 ops of the MMAs the kernel issued (device counters) / time;
    # peak = dense int8 tensor peak = 2 x the measured dense bf16 peak
    # (MEASURED_PEAKS.json, burst: the kernel is timed alone).
    cells_per_step = n_walks * n * (L - 1)
    per_step_s = (ms * 1e-3) / args.steps
    umma_ops = scan["umma"] * 128 * 64 * 32 * 2.0
    mma_ops = scan["mma"] * 16 * 8 * 32 * 2.0
    achieved = (umma_ops + mma_ops) / (ms * 1e-3)
    mp = measured_peaks()
    if mp.get("bf16_tflops"):
        peak = 2.0 * float(mp["bf16_tflops"]) * 1e12
        peak_src = ("2 x MEASURED_PEAKS.json bf16_tflops (burst, dense): the int8 tensor rate "
                    "is twice the bf16 rate")
    else:
        peak = 2.0 * 2250e12
        peak_src = "fallback: 2 x 2.25 PFLOP/s nominal dense bf16 (MEASURED_PEAKS.json absent)"
    traffic = None
    prof = os.path.join(ROOT, "profiles", "r02_cert_kernel.json")
    if os.path.exists(prof) and L == L_DEFAULT and n == 1024:
        try:
            pj = json.load(open(prof))
            # ncu --set full capture of run_kernel on this workload, scaled to one
            # step of this run's walk count
            traffic = pj["dram_bytes_per_launch"] / pj.get("steps_per_launch", 1) \
                * n_walks / float(pj.get("launch__grid_size", n_walks))
        except Exception:
            traffic = None
    int_roof = nsm * 64 * (mhz.value or 1965.0) * 1e6 / INT_OPS_PER_CELL
    roofline = {
        "bound": "tensor",
        "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "TOP/s (int8)",
        "frac": achieved / peak if peak else None,
        "traffic": traffic,
        "traffic_unit": "DRAM bytes per step (ncu --set full capture, profiles/r02_cert_kernel.json)",
        "algorithmic_bytes_per_step": n_walks * 8.0 * L,
        "peak_source": peak_src,
        "tcgen05_tops": umma_ops / (ms * 1e-3) / 1e12,
        "mma_sync_tops": mma_ops / (ms * 1e-3) / 1e12,
        "tcgen05_issue_peak_tops": (umma_per_s * 128 * 64 * 32 * 2.0 / 1e12) if umma_per_s else None,
        "frac_of_tcgen05_issue_peak": (achieved / (umma_per_s * 128 * 64 * 32 * 2.0))
        if umma_per_s else None,
        "mma_sync_peak_tops": (mma_per_s * 16 * 8 * 32 * 2.0 / 1e12) if mma_per_s else None,
        # tcgen05 (UMMA) and mma.sync (IMMA) serialise on the SM's tensor pipe
        # (profiles/r02_tensor_pipe_sharing.txt): the step's exclusive tensor-pipe
        # time at the probed rates (probe_umma walks the scan's descriptors)
        "tensor_pipe_busy_frac": ((scan["umma"] / umma_per_s + scan["mma"] / mma_per_s) / (ms * 1e-3))
        if (umma_per_s and mma_per_s) else None,
        "umma_per_step": scan["umma"] / args.steps,
        "mma_per_step": scan["mma"] / args.steps,
        "cells_per_s": cells_per_step / per_step_s,
        "cells_vs_int_roof": cells_per_step / per_step_s / int_roof,
        "int_roof_cells_per_s": int_roof,
        "fp64_dadd_peak_gcell_s": dadd.value / 1e9 if dadd.value else None,
        "probe_sm_mhz": mhz.value or None,
        "hbm_gbs_achieved": n_walks * 8.0 * L / per_step_s / 1e9,
        "scan_steps": {"certified": scan["certified"], "refined": scan["refined"],
                       "value_local_chains": scan["chains"]},
    }

    # the value-exact path: the same walks scored by the exact serial-chain sweep
    # (every neighbour's double bit-identical to detail::eval_flip)
    exact = None
    if args.exact_steps > 0:
        ctx.set_scan_mode(ctx.SCAN_EXACT)
        we = P.Walks(params(args.exact_steps + 2), n_walks, seeds=seeds, ctx=ctx)
        we.step(1)
        torch.cuda.synchronize()
        n0 = sum(r.nse for r in we.records())
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record(stream)
        we.step(args.exact_steps)
        eb.record(stream)
        torch.cuda.synchronize()
        ex_ms = D.max_over_ranks(ea.elapsed_time(eb), cdev)
        ex_nse = D.sum_over_ranks(float(sum(r.nse for r in we.records()) - n0), cdev)
        we.close()
        ctx.set_scan_mode(ctx.SCAN_AUTO)
        ex_value = ex_nse / (ex_ms * 1e-3)
        ex_cells = ex_value * (L - 1) / world
        exact = {"value": ex_value, "unit": "NSE/s", "steps": args.exact_steps,
                 "ms_per_step": ex_ms / args.exact_steps,
                 "scan": "exact (value-exact: every neighbour's serial double)",
                 "cells_per_s_per_gpu": ex_cells,
                 "frac_of_fp64_dadd_peak": ex_cells / dadd.value if dadd.value else None,
                 "frac_of_int_roof": ex_cells / int_roof}

    # e2e through the public API: host start sequences in, records + best
    # sequences out, table build + e2e_steps search steps inside the region
    rng = np.random.default_rng(1234 + rank)
    inits = np.where(rng.integers(0, 2, (n_walks, L)) == 1, -1, 1).astype(np.int8)
    inits_pinned = torch.from_numpy(inits).pin_memory().numpy()
    # the caller's pinned output buffer for the best sequences (reused per call)
    sol_pinned = torch.empty((n_walks, L), dtype=torch.int8).pin_memory().numpy()
    p2 = P.SearchParams(length=L, seed=args.seed, alpha1=4, alpha2=P.default_alpha2(L),
                        ls_lmt=2000, flip_lmt=min(L, 10), n_lmt=n,
                        stop=P.StopCondition(max_nse=1 + args.e2e_steps * n))
    # one untimed warm-up call (first-use pool growth), then e2e_reps timed calls
    P.run_walks(p2, n_walks, seeds=seeds, inits=inits_pinned, ctx=ctx, solutions=True,
                out=sol_pinned)
    torch.cuda.synchronize()
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_nse_local = 0.0
    if world > 1:
        dist.barrier()
    ea.record(stream)
    for _ in range(args.e2e_reps):
        recs = P.run_walks(p2, n_walks, seeds=seeds, inits=inits_pinned, ctx=ctx,
                           solutions=True, out=sol_pinned)
        e2e_nse_local += float(sum(r.nse for r in recs))
    eb.record(stream)
    torch.cuda.synchronize()
    e2e_ms = D.max_over_ranks(ea.elapsed_time(eb), cdev)
    e2e_nse = D.sum_over_ranks(e2e_nse_local, cdev)
    nwords = (L + 31) // 32
    e2e = {"value": e2e_nse / (e2e_ms * 1e-3), "unit": "NSE/s",
           "h2d_bytes_per_step": int(inits.nbytes + 8 * n_walks),
           "pcie_h2d_bytes_per_step": int(n_walks * nwords * 4 + 8 * n_walks),
           "d2h_bytes_per_step": int(n_walks * L + n_walks * 80),
           "steps": args.e2e_reps, "ms_per_step": e2e_ms / args.e2e_reps,
           "step": f"one psl_run_walks call per GPU: {n_walks} host start sequences (pinned "
                   f"int8, h2d_bytes_per_step) -> validated and bit-packed by the host threads, "
                   f"uploaded as bits (pcie_h2d_bytes_per_step) -> NTT table build + "
                   f"{args.e2e_steps} search steps -> records + best sequences (int8, into a "
                   f"pinned host buffer) on the host; 1 untimed warm-up call"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import oracle_py as O
            if O.ref_available():
                info = host_info()
                W, threads = reference_walks(L, n, args.seed)
                rate, secs, _ = W.step(args.cpu_steps)
                W.close()
                cpu = {"value": rate, "unit": "NSE/s", "cores": threads, "kind": "reference",
                       "sample": sample_desc(threads, L, n, args.cpu_steps, info),
                       "seconds": secs, "host": info}
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "NSE/s", "cores": os.cpu_count() or 1,
                   "kind": "reference", "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "NSE/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": max_ms / args.steps,
            "higher_is_better": True, "scaling": "weak",
            "vs_baseline": value / A100_M20_NSE,
            "dtype": "f64", "data": "synthetic",
            "scan": "certified (decision-exact: records, events, trajectories and best "
                    "sequences identical to the reference; neighbour doubles bracketed, "
                    "not computed -- see 'exact' for the value-exact sweep)",
            "config": {
                "workload": f"m20 two-phase search: L={L}, {n_walks} independent walks per GPU "
                            f"(one walk CTA per SM at a time, {-(-n_walks // nsm)} waves), "
                            f"alpha1=4, alpha2={P.default_alpha2(L)}, "
                            f"ls_lmt=2000, flip_lmt=10, n_lmt={n}",
                "L": L, "walks_per_gpu": n_walks, "n_lmt": n,
                "parallelism": f"walks x{world} (one process per GPU, {backend})",
                "l2": "inputs larger than L2: each step streams every walk's 4 MB C_k table "
                      f"({n_walks * 4 * L / 2**20:.0f} MiB per GPU per step) through L2",
                "vs_baseline_ref": "A100 solver 85062 NSE/s at L=1048575 (PAPER.md:342-359, "
                                   "N_lmt=6912)",
                "setup_seconds": setup_s},
            "cells_per_s": value * (L - 1),
            "roofline": roofline,
            "exact": exact,
            "clocks": clocks.summary(),
            "e2e": e2e,
            "gpu_launches": launches,
            "best_psl": best_psl, "best_walk": best_walk,
            "walk_records_sha": records_sha(rows),
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
