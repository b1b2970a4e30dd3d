"""Data-parallel plumbing for the hot path (host side only).

* ``shard_rows`` -- the row shard a rank owns (reading R13: ZeRO-2 averaged-gradient
  shards; contiguous, near-equal, remainder to the first ranks).
* ``flat_partition`` -- the row ranges a rank owns under a ZeRO-style flat partition
  (row f3): the model's gradients concatenated row-major and cut into
  ``world`` near-equal contiguous ranges, each boundary snapped to the nearest row start
  so that no row (and so no input channel's slice of a row) is split between ranks.
  Most matrices then live on one rank (n_local = 0 elsewhere, which ``zf_create``
  accepts); the ones straddling a boundary are split by rows.  The norm all-reduce sums
  the ranks' partial norms of every matrix as before.
* ``segment_map`` -- the (segment_id, offset) table of P:583 for such a partition: for
  each selected channel (segment_id = its slot) of each matrix this rank holds rows of,
  the offset of the channel's first element in the rank's flattened storage (stride m,
  n_local elements).
* ``broadcast_nccl_id`` -- rank 0 creates the 128-byte NCCL unique id through the
  C-ABI (``zf_nccl_unique_id``) and ``torch.distributed`` broadcasts it; every rank
  then passes it to ``zf_create`` (the norm all-reduce runs inside ``zf_step``).  One id
  per context.
* ``gloo_allreduce`` -- the host all-reduce callback (ranks without NCCL, e.g. sharing a GPU).
* ``open_peer_exchange`` -- the peer-memory exchange (f4 iii): all-gather the ranks' IPC
  handles, map them (``zf_peer_open``).
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
    """A fresh NCCL unique id from rank 0, broadcast to the group.  Call it once per
    ``zf.Context`` (an id bootstraps exactly one communicator), on every rank in the same
    order."""
    import torch.distributed as dist
    from . import zf
    obj = [zf.zf_nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def flat_partition(shapes, world: int, rank: int) -> list[tuple[int, int]]:
    """[start, stop) rows of every (n, m) matrix owned by `rank` under the row-snapped flat
    partition (see module doc).  Every row of every matrix belongs to exactly one rank."""
    if not (world >= 1 and 0 <= rank < world):
        raise ValueError("bad world/rank")
    offs = [0]
    for n, m in shapes:
        offs.append(offs[-1] + n * m)
    total = offs[-1]

    def snap(b: int) -> int:
        # element offset b -> the nearest row start (global flat offset)
        if b <= 0:
            return 0
        if b >= total:
            return total
        lo, hi = 0, len(shapes) - 1
        while lo < hi:                     # matrix holding element b
            mid = (lo + hi + 1) // 2
            if offs[mid] <= b:
                lo = mid
            else:
                hi = mid - 1
        n, m = shapes[lo]
        i, o = divmod(b - offs[lo], m)
        return offs[lo] + (i + (1 if 2 * o >= m else 0)) * m

    a = snap(rank * total // world)
    b = snap((rank + 1) * total // world)
    out = []
    for (n, m), o in zip(shapes, offs):
        r0 = min(n, max(0, -(-(a - o) // m)))
        r1 = min(n, max(0, -(-(b - o) // m)))
        out.append((r0, r1))
    return out


def segment_map(shapes, spans, idx_per_matrix):
    """P:583 segment mapping table for one rank: list of (matrix, segment_id, offset, stride,
    count) -- the selected channel idx[segment_id] of `matrix` occupies `count` elements at
    `offset`, `offset + stride`, ... of the rank's flattened (row-major) storage."""
    out, base = [], 0
    for li, ((n, m), (r0, r1), idx) in enumerate(zip(shapes, spans, idx_per_matrix)):
        rows = r1 - r0
        if rows > 0:
            for sid, c in enumerate(idx):
                out.append((li, sid, base + int(c), m, rows))
        base += rows * m
    return out


def gloo_allreduce(group=None):
    """A ``host_allreduce`` for ``zf.Context`` over a torch.distributed process group (e.g.
    gloo): sums the flat fp32 norm vector in place across the ranks (row a2 without NCCL)."""
    import torch
    import torch.distributed as dist

    def fn(buf):
        t = torch.from_numpy(buf)          # shares memory with the library's pinned buffer
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return fn


def open_peer_exchange(ctx, group=None):
    """Row a2 over peer memory (next row f4 (iii)): all-gather every rank's 64-byte
    IPC handle of its norm-exchange region over `group` (rank order) and map the others
    (``zf_peer_open``); the context's norm exchange then runs as kernels reading the peers'
    device memory (NVLink / NVSwitch, or one shared GPU), with no NCCL launch."""
    import torch.distributed as dist

    handles = [None] * dist.get_world_size(group)
    dist.all_gather_object(handles, ctx.peer_handle(), group=group)
    ctx.peer_open(handles)
