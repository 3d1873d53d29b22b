"""Host-side multi-GPU plumbing (one process per GPU, torch.distributed for the control plane).

The data path — per-sweep column partials exchanged with ncclAllGather and merged in
rank order — lives in the C library (sinkhorn_solve_sharded).  This module only:
  * computes the fixed row-block partition (sk_shard_rows) for every rank,
  * moves the 128-byte NCCL unique id from rank 0 to all ranks over the process group,
  * reduces host timings / counts across ranks (max of times, sum of work).
Everything here also runs on the gloo backend (CPU), which is how it is tested.
"""
from __future__ import annotations

import os
from typing import List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist

from . import shard_rows


def shard_plan(n_total: int, world: int) -> List[Tuple[int, int]]:
    """(row0, n_local) of every rank in the fixed partition (bit-identical across world sizes)."""
    return [shard_rows(n_total, r, world) for r in range(world)]


def exchange_unique_id(uid: Optional[bytes], group=None, src: int = 0) -> bytes:
    """Broadcast rank `src`'s 128-byte NCCL unique id to every rank of the group."""
    obj = [uid if dist.get_rank(group) == src else None]
    dist.broadcast_object_list(obj, src=src, group=group)
    out = obj[0]
    if not isinstance(out, (bytes, bytearray)) or len(out) != 128:
        raise RuntimeError("bad NCCL unique id broadcast")
    return bytes(out)


def init_comm(ctx, group=None) -> None:
    """Create the library's NCCL communicator over the same ranks as `group`."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = ctx.nccl_unique_id() if rank == 0 else None
    uid = exchange_unique_id(uid, group)
    ctx.comm_init(uid, rank, world)


def _reduce(vals: Sequence[float], op, device) -> List[float]:
    t = torch.tensor(list(vals), dtype=torch.float64, device=device)
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=op)
    return t.tolist()


def max_over_ranks(vals: Sequence[float], device="cpu") -> List[float]:
    return _reduce(vals, dist.ReduceOp.MAX, device)


def sum_over_ranks(vals: Sequence[float], device="cpu") -> List[float]:
    return _reduce(vals, dist.ReduceOp.SUM, device)


def env_rank() -> Tuple[int, int, int]:
    """(world, rank, local_rank) from the torchrun environment (1, 0, 0 if absent)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))
