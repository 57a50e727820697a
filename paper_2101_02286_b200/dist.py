"""torch.distributed plumbing for multi-GPU plans (one process per GPU).

Only host-side logic lives here: rank 0 draws the NCCL unique id through the
C ABI and broadcasts the 128 bytes over the caller's process group (NCCL or
gloo); every rank then creates its plan.  The solve itself never touches
torch.distributed -- the library's own NCCL communicator carries the
reduced-system messages.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import ctri


def broadcast_unique_id(make_id=None, group=None, src: int = 0) -> bytes:
    """Rank `src` creates a 128-byte id (``make_id()``, default ctri_get_unique_id) and every
    rank of `group` returns the same bytes."""
    make_id = make_id or ctri.ctri_get_unique_id
    obj = [make_id() if dist.get_rank(group) == src else None]
    dist.broadcast_object_list(obj, src=src, group=group)
    uid = obj[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise RuntimeError("bad NCCL unique id received")
    return bytes(uid)


def plan_from_process_group(global_dims, solve_dim=0, bands=(1 / 3, 1.0, 1 / 3), cyclic=True,
                            flags=0, group=None, stream=None) -> ctri.Plan:
    """Collective: one plan per rank, nparts = world size, rank = group rank."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    uid = broadcast_unique_id(group=group) if world > 1 else None
    return ctri.Plan(global_dims, solve_dim, world, rank, bands, cyclic, uid, flags, stream)


def slab_bounds(N: int, nparts: int, rank: int):
    """Rows [lo, hi) of the solve direction owned by `rank` (equal split, P:5)."""
    if N % nparts:
        raise ValueError("N must be divisible by nparts")
    n = N // nparts
    return rank * n, (rank + 1) * n


def gather_to_rank0(local: torch.Tensor, solve_dim: int, group=None):
    """Gather every rank's slab (same shape) to rank 0 and concatenate along solve_dim."""
    world = dist.get_world_size(group)
    if world == 1:
        return local
    parts = [torch.empty_like(local) for _ in range(world)] if dist.get_rank(group) == 0 else None
    dist.gather(local.contiguous(), parts, dst=0, group=group)
    if dist.get_rank(group) == 0:
        return torch.cat(parts, dim=solve_dim)
    return None


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank float (timings are reported as the max over ranks)."""
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
