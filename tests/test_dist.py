"""Multi-process (gloo, world_size 2, CPU) tests of the end-of-run reduction:
walks shard across ranks with no per-step traffic; at the end the best PSL
(ties -> smaller global walk id) is all-reduced and its sequence broadcast.
This is the collective bench.py runs over NCCL on N GPUs."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2107_09801_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, L, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(100 + rank)
    W = 3
    ids = [rank * W + w for w in range(W)]
    sols = [np.where(rng.integers(0, 2, L) == 1, -1, 1).astype(np.int8) for _ in ids]
    # rank 1 holds the global best (psl 7) twice; the smaller id must win
    psls = [9, 11, 12] if rank == 0 else [7, 7, 10]
    psl, wid, sol = D.reduce_best(psls, ids, sols, L)
    mx = D.max_over_ranks(float(rank + 1))
    sm = D.sum_over_ranks(float(rank + 1))
    out.put((rank, psl, wid, sol.tobytes(), mx, sm,
             sols[0].tobytes() if rank == 1 else None))
    dist.destroy_process_group()


def test_reduce_best_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    L = 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, L, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    winner_sol = res[1][6]
    for rank, psl, wid, sol, mx, sm, _ in res:
        assert (psl, wid) == (7, 3)          # rank 1, local index 0 -> global id 3
        assert sol == winner_sol
        assert (mx, sm) == (2.0, 3.0)


def test_pack_roundtrip_and_keys():
    rng = np.random.default_rng(0)
    for L in (2, 7, 8, 9, 1000, 1048575):
        s = np.where(rng.integers(0, 2, L) == 1, -1, 1).astype(np.int8)
        assert np.array_equal(D.unpack_bits(D.pack_bits(s), L), s)
    assert D.unpack_key(D.pack_key(901, 1183)) == (901, 1183)
    assert D.pack_key(5, 9) < D.pack_key(5, 10) < D.pack_key(6, 0)
    key, idx = D.local_best([4, 3, 3], [10, 12, 11])
    assert (key >> 32, key & 0xffffffff, idx) == (3, 11, 2)


def _bench(args, env=None, timeout=300):
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(root, "bench.py")] + args,
                          capture_output=True, text=True, timeout=timeout, env=e, cwd=root)


def test_bench_gpus_n_launches_n_ranks():
    """bench.py --gpus 2 started directly re-launches itself under
    torch.distributed.run with 2 processes; the reference arm runs on rank 0
    only and prints exactly one JSON line (the other rank exits 0)."""
    import json
    from oracle import oracle_py as O
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    p = _bench(["--impl", "reference", "--gpus", "2", "--length", "4095", "--steps", "2",
                "--warmup", "1"])
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["value"] > 0
    assert line["cpu_baseline"]["cores"] == line["config"]["host_threads"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_bench_rejects_world_mismatch():
    p = _bench(["--impl", "reference", "--gpus", "1", "--length", "64"],
               env={"WORLD_SIZE": "2", "RANK": "1", "LOCAL_RANK": "1"})
    assert p.returncode == 2 and "world size 2 != --gpus 1" in p.stderr
