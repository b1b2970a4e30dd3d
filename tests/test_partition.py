"""Flat ZeRO-style partitions (row f3) -- host logic, CPU only:
row-snapped flat partition of the concatenated row-major gradients, the segment map of
P:583, and (world size 2 over gloo) the norm exchange on such a partition."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from paper_2505_12242_b200.dist import flat_partition, segment_map

SHAPES = [(37, 1001), (513, 768), (130, 257), (5, 2000), (1, 64), (64, 4096), (250, 130)]


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8, 13])
def test_flat_partition_covers_every_row_once(world):
    spans = [flat_partition(SHAPES, world, r) for r in range(world)]
    for li, (n, m) in enumerate(SHAPES):
        owned = np.zeros(n, np.int32)
        for r in range(world):
            a, b = spans[r][li]
            assert 0 <= a <= b <= n
            owned[a:b] += 1
        assert np.all(owned == 1), (li, owned)
    # ranks hold consecutive flat ranges, in rank order
    flat = []
    offs = np.cumsum([0] + [n * m for n, m in SHAPES])
    for r in range(world):
        ranges = [(offs[li] + a * m, offs[li] + b * m) for li, ((a, b), (n, m)) in enumerate(zip(spans[r], SHAPES))
                  if b > a]
        if ranges:
            for (x0, x1), (y0, y1) in zip(ranges, ranges[1:]):
                assert x1 == y0
            flat.append((ranges[0][0], ranges[-1][1]))
    for (x0, x1), (y0, y1) in zip(flat, flat[1:]):
        assert x1 == y0
    assert flat[0][0] == 0 and flat[-1][1] == offs[-1]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_flat_partition_balance(world):
    """Each boundary moves by at most half a row from the exact equal split."""
    shapes = [(n, m) for _, n, m in synth.llama2_7b_linears()]
    total = sum(n * m for n, m in shapes)
    for r in range(world):
        own = sum((b - a) * m for (a, b), (n, m) in zip(flat_partition(shapes, world, r), shapes))
        assert abs(own - total / world) <= 11008 + 1


def test_segment_map_reassembles_channels():
    """reassembled channel slices equal the unsharded column."""
    rng = np.random.default_rng(5)
    world = 3
    mats = [rng.standard_normal((n, m)).astype(np.float32) for n, m in SHAPES]
    idxs = [np.sort(rng.choice(m, size=max(1, m // 10), replace=False)).astype(np.int32) for n, m in SHAPES]
    got = [[[] for _ in idx] for idx in idxs]
    for r in range(world):
        spans = flat_partition(SHAPES, world, r)
        store = np.concatenate([mats[li][a:b].reshape(-1) for li, (a, b) in enumerate(spans)])
        for li, sid, off, stride, cnt in segment_map(SHAPES, spans, idxs):
            got[li][sid].append(store[off:off + stride * cnt:stride])
    for li, idx in enumerate(idxs):
        for sid, c in enumerate(idx):
            assert np.array_equal(np.concatenate(got[li][sid]), mats[li][:, c])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    from oracle import oracle as orc
    spans = flat_partition(SHAPES, world, rank)
    sel = []
    for li, ((n, m), (a, b)) in enumerate(zip(SHAPES, spans)):
        e = synth.col_scale_init(m, layer=li)
        G = synth.grad(b - a, m, layer=li, step=0, scale_exp=e, dtype="fp32", row0=a)
        part = torch.from_numpy(orc.column_norms(G))       # zeros when the rank holds no rows
        dist.all_reduce(part, op=dist.ReduceOp.SUM)
        sel.append(orc.topk(part.numpy(), orc.k_for(m, 100000)))
        np.save(os.path.join(out_dir, f"norms_{rank}_{li}.npy"), part.numpy())
    np.save(os.path.join(out_dir, f"sel_{rank}.npy"), np.concatenate(sel))
    dist.destroy_process_group()


def test_flat_partition_norm_exchange_gloo(tmp_path):
    """world 2, flat partition: the all-reduced partial norms of every matrix equal the
    unsharded oracle norms (rel 1e-6), and both ranks select the same columns."""
    from oracle import oracle as orc
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for li, (n, m) in enumerate(SHAPES):
        G = synth.grad(n, m, layer=li, step=0, scale_exp=synth.col_scale_init(m, layer=li), dtype="fp32")
        want = orc.column_norms(G).astype(np.float64)
        for r in range(world):
            got = np.load(tmp_path / f"norms_{r}_{li}.npy").astype(np.float64)
            assert np.all(np.abs(got - want) <= 1e-6 * np.abs(want) + 1e-30), li
    assert np.array_equal(np.load(tmp_path / "sel_0.npy"), np.load(tmp_path / "sel_1.npy"))


def test_flat_partition_snaps_to_the_nearest_row():
    """Worked example of the row snapping (module doc of dist.flat_partition): one 10x100
    matrix over 3 ranks has element boundaries 333 and 666, which snap to the nearest row
    starts 300 (33 past a row start) and 700 (34 before one): rows [0,3), [3,7), [7,10).
    Two matrices [(4, 10), (6, 10)] over 2 ranks: boundary 50 = row 1 of the second matrix."""
    from paper_2505_12242_b200.dist import flat_partition
    assert [flat_partition([(10, 100)], 3, r) for r in range(3)] == [[(0, 3)], [(3, 7)], [(7, 10)]]
    assert [flat_partition([(4, 10), (6, 10)], 2, r) for r in range(2)] == [[(0, 4), (0, 1)], [(4, 4), (1, 6)]]
