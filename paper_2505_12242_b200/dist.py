"""Data-parallel plumbing for the hot path (host side only).

* ``shard_rows`` -- the row shard a rank owns (reading R13: ZeRO-2 averaged-gradient
  shards; contiguous, near-equal, remainder to the first ranks).
* ``broadcast_nccl_id`` -- rank 0 creates the 128-byte NCCL unique id through the
  C-ABI (``zf_nccl_unique_id``) and ``torch.distributed`` broadcasts it; every rank
  then passes it to ``zf_create`` (the norm all-reduce runs inside ``zf_step``).
"""
from __future__ import annotations


def shard_rows(n: int, world: int, rank: int) -> tuple[int, int]:
    """[start, stop) rows of an n-row matrix owned by `rank` of `world`."""
    if not (world >= 1 and 0 <= rank < world):
        raise ValueError("bad world/rank")
    base, rem = divmod(n, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


def broadcast_nccl_id(group=None) -> bytes:
    import torch.distributed as dist
    from . import zf
    obj = [zf.zf_nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]
