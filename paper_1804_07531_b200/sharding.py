"""Host-side helpers for the row-sharded multi-GPU path (one process per GPU).

The library (librsvd) shards A by contiguous row blocks: rank r holds rows [row0, row0 + m_local).
  * A X        (range view)     : local on every rank, the result stays row-sharded
  * A^T Y      (co-range view)  : each rank computes its partial A_r^T Y_r, NCCL all-reduce
  * Gram / cross products of row-sharded blocks (orthonormalisation, Phi^T Q_c): all-reduce
  * everything on the column side (n rows: Q_r, Z, V) is replicated and bitwise identical
These helpers plan the shards, exchange the NCCL unique id through a torch process group and take
maxima over ranks for timing; they hold no arithmetic of the method.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    m: int          # global rows
    row0: int
    m_local: int


def shard_rows(m: int, world: int, rank: int, align: int = 1) -> Shard:
    """Contiguous row blocks in rank order that tile [0, m): the first (m // align) % world blocks
    get one extra `align`-sized chunk.  Every rank gets at least one row when m >= world."""
    if world < 1 or not (0 <= rank < world) or m < world:
        raise ValueError("need world >= 1, 0 <= rank < world and m >= world")
    chunks = -(-m // align)
    base, extra = divmod(chunks, world)
    c0 = rank * base + min(rank, extra)
    c1 = c0 + base + (1 if rank < extra else 0)
    row0 = min(m, c0 * align)
    row1 = min(m, c1 * align)
    return Shard(rank, world, m, row0, row1 - row0)


def weak_scaled(m_per_rank: int, world: int, rank: int) -> Shard:
    """Weak scaling: every rank holds an m_per_rank block of a (world * m_per_rank)-row matrix."""
    return Shard(rank, world, m_per_rank * world, m_per_rank * rank, m_per_rank)


def broadcast_uid(uid_on_rank0: bytes | None, rank: int, group=None) -> bytes:
    """Rank 0's 128-byte NCCL unique id to every rank (torch.distributed object broadcast)."""
    import torch.distributed as dist

    obj = [uid_on_rank0 if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    uid = obj[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise RuntimeError("bad NCCL unique id")
    return bytes(uid)


def max_over_ranks(x: float, device=None, group=None) -> float:
    """Max of a scalar over all ranks (multi-GPU timings are the slowest rank's)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
