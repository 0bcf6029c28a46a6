#!/usr/bin/env python
"""Benchmark: flip-evaluations/s (NSE/s) of the two-phase low-PSL search at
L = 2^20 - 1 (BASELINE.json metric), one JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step = one search step of every walk on every GPU: each walk scans its
n_lmt = 1024 one-flip neighbours (1024 x (L-1) flip x shift cells), reduces,
moves (and restarts when the phase rule fires), all on the device.  Walks are
independent (seed = seed0 + global walk id), one CTA per SM, so per-GPU work is
fixed as N grows ("scaling": "weak").  Inputs are synthetic random start
sequences (random_sequence(L, Rng(seed))), the reference's own start.

--impl reference times the reference's CPU implementation of the same path
(oracle/_ref/libpslref.so, compiled from the unmodified reference sources) on
all host cores: each step, every host thread scores the 1024 one-flip
neighbours of an L = 2^20 - 1 pivot with the reference's detail::eval_flip.
"""
from __future__ import annotations

import argparse
import json
import os
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
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
    ap.add_argument("--cpu-reps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


# ---------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

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

def reference_sample(L: int, n: int, reps: int, threads: int, seed: int):
    """The reference's own kernel (detail::eval_flip) on all host threads:
    each thread scores n neighbours of an L pivot `reps` times.  Returns
    (NSE/s, seconds, description).  The pivot's table comes from the oracle's
    threaded bit-parallel build (setup, untimed)."""
    from oracle import oracle_py as O
    R = O.ref()
    s = O.random_sequence(seed, L)
    c = O.build_table(s, threads=threads)
    lut = O.power_table(L + 4, 4)
    secs = C_double()
    rate = R.ref_bench_eval(s, c, L, 1, lut, n, reps, threads, secs)
    desc = (f"{threads} host threads x {reps} x {n} one-flip neighbour evaluations "
            f"(reference detail::eval_flip, sequence.hpp:126-162) of an L={L} random pivot, "
            f"alpha=4; table built by the oracle (untimed)")
    return rate, secs.value, desc


def C_double():
    import ctypes
    return ctypes.c_double()


def run_reference_arm(args, rank: int):
    if rank != 0:
        return
    from oracle import oracle_py as O
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libpslref.so not built (needs /root/reference at build time)"}))
        return
    L, n = args.length, args.n_lmt
    threads = os.cpu_count() or 1
    R = O.ref()
    s = O.random_sequence(args.seed, L)
    c = O.build_table(s, threads=threads)
    lut = O.power_table(L + 4, 4)
    secs = C_double()
    for _ in range(args.warmup):
        R.ref_bench_eval(s, c, L, 1, lut, n, 1, threads, secs)
    total = 0.0
    for _ in range(args.steps):
        R.ref_bench_eval(s, c, L, 1, lut, n, 1, threads, secs)
        total += secs.value
    nse = float(threads) * n * args.steps
    value = nse / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "NSE/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": value / A100_M20_NSE, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"m20: L={L}, {threads} walks (one per host core), n_lmt={n}",
                   "L": L, "n_lmt": n, "host_threads": threads,
                   "step": "every host thread scores the n one-flip neighbours of its pivot"},
        "cpu_baseline": {"value": value, "unit": "NSE/s", "cores": threads, "kind": "reference",
                         "sample": f"{threads} threads x {n} eval_flip per step, L={L}"},
        "e2e": {"value": value, "unit": "NSE/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "cells_per_s": value * (L - 1),
    }
    print(json.dumps(line))


# ---------------------------------------------------------------- ours

def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank)
        return

    import torch
    import torch.distributed as dist

    import paper_2107_09801_b200 as P
    from paper_2107_09801_b200 import dist as D

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    ctx = P.Context(local_rank)
    # a dedicated (non-default) stream shared by the engine and the CUDA events
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    nsm = torch.cuda.get_device_properties(local_rank).multi_processor_count
    # one 512-thread walk CTA per SM at a time (~211 KB smem); three waves of
    # walks per launch: a CTA that finishes its K steps early hands its SM to the
    # next walk (measured: 148 walks 24.0, 296 25.1, 444 25.6 M NSE/s)
    n_walks = args.walks or 3 * nsm
    L, n = args.length, args.n_lmt
    total_steps = args.warmup + args.steps + 4
    params = P.SearchParams(length=L, seed=args.seed, alpha1=4, alpha2=P.default_alpha2(L),
                            ls_lmt=2000, flip_lmt=min(L, 10), n_lmt=n,
                            stop=P.StopCondition(max_nse=1 + total_steps * (n + 1)))
    seeds = [args.seed + rank * n_walks + w for w in range(n_walks)]

    # roofline denominators measured on this GPU, now
    import ctypes
    dadd, lds, mhz = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    err = ctypes.create_string_buffer(256)
    P._lib.lib().psl_probe_peaks(ctx.handle, ctypes.byref(dadd), ctypes.byref(lds),
                                 ctypes.byref(mhz), err, 256)
    mma_per_s = ctx.probe_imma()
    umma_per_s = ctx.probe_umma()

    # setup: pivots (random_sequence), O(L^2) tables -- untimed, like the reference
    t_setup = time.perf_counter()
    walks = P.Walks(params, n_walks, seeds=seeds, ctx=ctx)
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
    with ClockSampler(local_rank) as clocks:
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
    max_ms = D.max_over_ranks(ms, dev)
    nse_total = D.sum_over_ranks(float(nse_local), dev)
    value = nse_total / (max_ms * 1e-3)
    # end-of-run best-PSL reduction across GPUs (outside the timed region)
    best_psl, best_walk, _ = D.reduce_best([r.psl_best for r in r1], seeds,
                                           [r.solution_best for r in r1], L, device=dev)
    walks.close()

    # dominant kernel: run_kernel, one launch for the K timed steps.  Steps are
    # scored by the certified scan: the correlation on tcgen05
    # (kind::i8 M128 N64 K32, accumulators in TMEM), the zone-1 cross term on
    # mma.sync m16n8k32, the exact DADD sweep only where intervals cannot decide.
    # achieved = int8 ops of the MMAs the kernel issued (device counters) / time;
    # peak = the tcgen05 kind::i8 instruction's measured issue rate on this GPU.
    cells_per_step = n_walks * n * (L - 1)
    per_step_s = (ms * 1e-3) / args.steps
    umma_ops = scan["umma"] * 128 * 64 * 32 * 2.0
    mma_ops = scan["mma"] * 16 * 8 * 32 * 2.0
    achieved = (umma_ops + mma_ops) / (ms * 1e-3)
    peak = umma_per_s * 128 * 64 * 32 * 2.0
    traffic = None
    prof = os.path.join(ROOT, "profiles", "r01_cert_kernel.json")
    if os.path.exists(prof) and L == L_DEFAULT and n == 1024:
        try:
            pj = json.load(open(prof))
            # ncu --set full capture of run_kernel on this workload, scaled to one
            # step of this run's walk count (profiles/r01_cert_kernel.txt)
            traffic = pj["dram_bytes_per_launch"] / pj.get("steps_per_launch", 1) \
                * n_walks / float(pj.get("launch__grid_size", n_walks))
        except Exception:
            traffic = None
    roofline = {
        "bound": "tensor",
        "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "TOP/s (int8)",
        "frac": achieved / peak if peak else None,
        "traffic": traffic,
        "traffic_unit": "DRAM bytes per step (ncu capture, profiles/r01_cert_kernel.json)",
        "algorithmic_bytes_per_step": n_walks * 8.0 * L,
        "peak_source": "measured live: tcgen05.mma kind::i8 M128 N64 K32 issue rate of this GPU "
                       "(psl_probe_umma); the kernel's MMAs are counted on the device",
        "tcgen05_tops": umma_ops / (ms * 1e-3) / 1e12,
        "mma_sync_tops": mma_ops / (ms * 1e-3) / 1e12,
        "mma_sync_peak_tops": mma_per_s * 16 * 8 * 32 * 2.0 / 1e12,
        "umma_per_step": scan["umma"] / args.steps,
        "mma_per_step": scan["mma"] / args.steps,
        "cells_per_s": cells_per_step / per_step_s,
        "fp64_dadd_peak_gcell_s": dadd.value / 1e9,
        "probe_sm_mhz": mhz.value,
        "hbm_gbs_achieved": n_walks * 8.0 * L / per_step_s / 1e9,
        "scan_steps": {"certified": scan["certified"], "refined": scan["refined"],
                       "value_local_chains": scan["chains"]},
    }

    # e2e through the public API: host start sequences in, records + best
    # sequences out, table build + e2e_steps search steps inside the region
    e2e = None
    if rank == 0 or True:
        rng = np.random.default_rng(1234 + rank)
        inits = np.where(rng.integers(0, 2, (n_walks, L)) == 1, -1, 1).astype(np.int8)
        inits_t = torch.from_numpy(inits).pin_memory()
        inits_pinned = inits_t.numpy()
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
        ea.record(stream)
        for _ in range(args.e2e_reps):
            recs = P.run_walks(p2, n_walks, seeds=seeds, inits=inits_pinned, ctx=ctx,
                               solutions=True, out=sol_pinned)
            e2e_nse_local += float(sum(r.nse for r in recs))
        eb.record(stream)
        torch.cuda.synchronize()
        e2e_ms = D.max_over_ranks(ea.elapsed_time(eb), dev)
        e2e_nse = D.sum_over_ranks(e2e_nse_local, dev)
        e2e = {"value": e2e_nse / (e2e_ms * 1e-3), "unit": "NSE/s",
               "h2d_bytes_per_step": int(inits.nbytes + 8 * n_walks),
               "d2h_bytes_per_step": int(n_walks * L + n_walks * 80),
               "steps": args.e2e_reps, "ms_per_step": e2e_ms / args.e2e_reps,
               "step": f"one psl_run_walks call: {n_walks} host start sequences (pinned int8) -> "
                       f"device validation/packing + NTT table build + {args.e2e_steps} search "
                       f"steps -> records + best sequences (int8, into a pinned host buffer) on the host; "
                       f"1 untimed warm-up call"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import oracle_py as O
            if O.ref_available():
                rate, secs, desc = reference_sample(L, n, args.cpu_reps, os.cpu_count() or 1,
                                                    args.seed)
                cpu = {"value": rate, "unit": "NSE/s", "cores": os.cpu_count() or 1,
                       "kind": "reference", "sample": desc, "seconds": secs}
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
            "config": {
                "workload": f"m20 two-phase search: L={L}, {n_walks} independent walks per GPU "
                            f"(one walk CTA per SM at a time, {-(-n_walks // nsm)} waves), "
                            f"alpha1=4, alpha2={P.default_alpha2(L)}, "
                            f"ls_lmt=2000, flip_lmt=10, n_lmt={n}",
                "L": L, "walks_per_gpu": n_walks, "n_lmt": n, "parallelism": f"walks x{world}",
                "l2": "inputs larger than L2: each step streams every walk's 4 MB C_k table "
                      f"({n_walks * 4 * L / 2**20:.0f} MiB per GPU per step) through L2",
                "vs_baseline_ref": "A100 solver 85062 NSE/s at L=1048575 (PAPER.md:342-359, "
                                   "N_lmt=6912)",
                "setup_seconds": setup_s},
            "cells_per_s": value * (L - 1),
            "roofline": roofline,
            "clocks": clocks.summary(),
            "e2e": e2e,
            "gpu_launches": launches,
            "best_psl": best_psl, "best_walk": best_walk,
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
