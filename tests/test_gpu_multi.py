"""New C-ABI entry points on the device, and the many-GPU path.

* psl_flip_deltas (sequence.cpp:154-172) and psl_fitness (sequence.cpp:131-141)
  against the pinned CPU oracle, bit for bit, at small and BASELINE lengths.
* psl_run_walks_multi: walks split over several device contexts (one host
  thread each; here two contexts on the one B200 of the box) give the same
  per-walk records and best sequences as one psl_run_walks over all walks, and
  the host-gathered winner is the (psl_best, walk index) minimum.
* bench.py's rank path: two processes (gloo rendezvous, one context each on
  cuda:0) shard the walk seeds exactly like the N-GPU bench and reproduce the
  single-process result; the walks are independent, so nothing waits on a peer.
"""
import ctypes as C
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle_py as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _oracle_deltas(s, j):
    out = np.zeros(len(s), np.int32)
    O.lib().orc_flip_deltas(s, len(s), j, out)
    return out


@pytest.mark.parametrize("L", [2, 3, 31, 64, 257, 4095, 65535, 1048575])
def test_flip_deltas_match_oracle(engine, L):
    rng = np.random.default_rng(L)
    s = rng.choice(np.array([-1, 1], np.int8), L)
    for j in sorted({0, L - 1, L // 2, int(rng.integers(0, L))}):
        d = engine.flip_deltas(s, j)
        assert np.array_equal(d, _oracle_deltas(s, j)), (L, j)
        # apply_flip == table + deltas (sequence.hpp:93-97)
        if L <= 4095:
            c = O.build_table(s)
            s2 = s.copy()
            s2[j] = -s2[j]
            assert np.array_equal(O.build_table(s2)[1:], (c + d)[1:])
    with pytest.raises(engine.ConfigError, match="out of range"):
        engine.flip_deltas(s, L)


@pytest.mark.parametrize("L,alphas", [(13, (1, 2, 4)), (300, (1, 4, 13)), (4095, (4, 13)),
                                      (65535, (4, 13)), (262143, (4, 11)), (1048575, (4, 10))])
def test_device_fitness_chain_matches_oracle(engine, L, alphas):
    s = O.random_sequence(1, L)
    c = O.build_table(s, fast=True)
    for a in alphas:
        lut = O.power_table(L, a)
        f = engine.fitness(c, engine.PowerTable(L, a))
        assert f.hex() == O.fitness(c, lut).hex(), (L, a)
    assert engine.fitness(c, 4) == engine.fitness(c, engine.PowerTable(L, 4))


def test_fitness_overflow_and_psl_mf(engine, golden):
    ones = np.ones(64, np.int8)
    c = O.build_table(ones)
    with pytest.raises(engine.OverflowError, match="fitness sum is not finite at length 64"):
        engine.fitness(c, 1100)
    # the m14 KAT's initial fitness, host psl / merit factor
    g = golden("kats.json")["16383"]
    s = O.random_sequence(1, 16383)
    c = O.build_table(s, fast=True)
    assert engine.fitness(c, 4).hex() == g["initial_fitness"]
    assert engine.psl(c) == g["initial_psl"]


def _params(engine, L, n, steps, seed=1, a2=None):
    return engine.SearchParams(length=L, seed=seed, alpha1=4,
                               alpha2=a2 if a2 else engine.default_alpha2(L), ls_lmt=3,
                               flip_lmt=min(L, 10), n_lmt=n,
                               stop=engine.StopCondition(max_nse=1 + steps * n))


@pytest.mark.parametrize("L,walks,steps", [(4095, 7, 60), (65535, 5, 12)])
def test_run_walks_multi_equals_single(engine, L, walks, steps):
    p = _params(engine, L, min(L, 1024), steps)
    seeds = [100 + 3 * w for w in range(walks)]
    one = engine.run_walks(p, walks, seeds=seeds)
    multi, best, secs = engine.run_walks_multi(p, walks, devices=[0, 0], seeds=seeds)
    assert len(secs) == 2 and all(x > 0 for x in secs)
    for a, b in zip(one, multi):
        assert (a.seed, a.nse, a.psl_best, a.energy, a.switches, a.steps) == \
            (b.seed, b.nse, b.psl_best, b.energy, b.switches, b.steps)
        assert np.array_equal(a.solution_best, b.solution_best)
    key = min((r.psl_best, i) for i, r in enumerate(one))
    assert best == key[1]
    # walk w of the multi run is run_search(seed_w): the reference's own record
    rc, o, osol, _, _ = O.run_search(L, seeds[best], 4, engine.default_alpha2(L), 3, 10,
                                     min(L, 1024), 1 + steps * min(L, 1024), traces_cap=0)
    assert rc == 0 and o.psl_best == multi[best].psl_best
    assert np.array_equal(osol, multi[best].solution_best)


def test_run_walks_multi_errors(engine):
    p = _params(engine, 64, 16, 5)
    with pytest.raises(engine.ConfigError, match="number of devices"):
        engine.run_walks_multi(p, 1, devices=[0, 0])
    with pytest.raises(engine.DeviceError, match="device 99"):
        engine.run_walks_multi(p, 2, devices=[0, 99])


def test_bench_rank_path_two_processes(tmp_path):
    """bench.py --gpus 2 under a 2-process gloo launch on one GPU (both ranks on
    cuda:0 via PSLB200_BENCH_SAME_DEVICE): n_gpus 2, sharded seeds, and the
    host-reduced best PSL equals a single process running all the walks."""
    env = dict(os.environ, PSLB200_BENCH_SAME_DEVICE="1", PSLB200_BENCH_BACKEND="gloo")
    args = ["--length", "65535", "--walks", "4", "--steps", "3", "--warmup", "3",
            "--e2e-reps", "1", "--e2e-steps", "2", "--no-cpu-baseline", "--no-probes"]
    two = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"] + args,
                         capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert two.returncode == 0, two.stdout[-3000:] + two.stderr[-3000:]
    line = json.loads([ln for ln in two.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["config"]["walks_per_gpu"] == 4
    # rank r ran seeds 1 + 4r .. 4r + 4: the same 8 walks in one process
    one = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "1",
                          "--length", "65535", "--walks", "8", "--steps", "3", "--warmup", "3",
                          "--e2e-reps", "1", "--e2e-steps", "2", "--no-cpu-baseline",
                          "--no-probes"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert one.returncode == 0, one.stderr[-3000:]
    l1 = json.loads([ln for ln in one.stdout.splitlines() if ln.startswith("{")][-1])
    assert (line["best_psl"], line["best_walk"]) == (l1["best_psl"], l1["best_walk"])
    assert line["walk_records_sha"] == l1["walk_records_sha"]
