"""Multi-GPU plumbing: independent walks per rank, end-of-run best-PSL argmin.

The search shards as independent walks: rank r runs walks
with global ids r*W .. r*W+W-1 (seed = seed0 + global id) and there is no
per-step communication.  The only collective is at the end: an all-reduce MIN
of the packed key (psl_best << 32) | global_walk_id -- ties resolve to the
smaller walk id -- followed by a broadcast of the owner's sequence (bit-packed,
<= 128 KiB).  Works with NCCL (tensors on the rank's GPU) and with gloo (CPU
tensors; used by the world_size-2 tests).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def pack_key(psl_best: int, walk_id: int) -> int:
    return (int(psl_best) << 32) | int(walk_id)


def unpack_key(key: int) -> tuple[int, int]:
    return key >> 32, key & 0xffffffff


def pack_bits(seq: np.ndarray) -> np.ndarray:
    bits = (np.asarray(seq) < 0).astype(np.uint8)
    return np.packbits(bits, bitorder="little")


def unpack_bits(packed: np.ndarray, length: int) -> np.ndarray:
    bits = np.unpackbits(packed, bitorder="little")[:length]
    return np.where(bits == 1, -1, 1).astype(np.int8)


def local_best(psls, walk_ids) -> tuple[int, int]:
    """Smallest psl_best, ties to the smallest global walk id."""
    best = min(pack_key(p, w) for p, w in zip(psls, walk_ids))
    return best, walk_ids.index(best & 0xffffffff)


def reduce_best(psls, walk_ids, solutions, length: int, device=None):
    """Returns (psl_best, global_walk_id, solution) identical on every rank.

    psls/walk_ids/solutions describe this rank's walks (solutions[i] is the
    int8 +-1 sequence of walk_ids[i])."""
    key, idx = local_best(list(psls), list(walk_ids))
    dev = device if device is not None else torch.device("cpu")
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return key >> 32, key & 0xffffffff, np.asarray(solutions[idx], np.int8)
    t = torch.tensor([key], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    gkey = int(t.item())
    mine = gkey == key
    owner = torch.tensor([dist.get_rank() if mine else 1 << 30], dtype=torch.int64, device=dev)
    dist.all_reduce(owner, op=dist.ReduceOp.MIN)
    src = int(owner.item())
    nbytes = (length + 7) // 8
    buf = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
    if dist.get_rank() == src:
        buf.copy_(torch.from_numpy(pack_bits(solutions[idx])).to(dev))
    dist.broadcast(buf, src=src)
    sol = unpack_bits(buf.cpu().numpy(), length)
    return gkey >> 32, gkey & 0xffffffff, sol


def max_over_ranks(value: float, device=None) -> float:
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device or torch.device("cpu"))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device or torch.device("cpu"))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
