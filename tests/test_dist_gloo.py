"""World-size-2 data-parallel protocol on CPU (gloo): row shards, NCCL-id bootstrap
through torch.distributed, and the norm exchange of P:486 -- summing the ranks'
partial column norms reproduces the unsharded norms, and every rank then selects the
same columns."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


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
    import synth
    from oracle import oracle as orc
    from paper_2505_12242_b200 import dist as zdist
    nid = zdist.broadcast_nccl_id()
    n, m = 1030, 700
    e = synth.col_scale_init(m, layer=3)
    r0, r1 = zdist.shard_rows(n, world, rank)
    G = synth.grad(r1 - r0, m, layer=3, step=0, scale_exp=e, dtype="fp32", row0=r0)
    part = torch.from_numpy(orc.column_norms(G))
    zdist.gloo_allreduce()(part.numpy())          # the product's host all-reduce callback (in place)
    k = orc.k_for(m, 100000)
    idx = orc.topk(part.numpy(), k)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), nid=np.frombuffer(nid, np.uint8), norms=part.numpy(),
             idx=idx, rows=np.array([r0, r1]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_norm_exchange(tmp_path):
    from paper_2505_12242_b200 import _build
    _build.build()
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    res = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    import synth
    from oracle import oracle as orc
    # same NCCL id on both ranks; shards tile the rows
    assert np.array_equal(res[0]["nid"], res[1]["nid"]) and len(res[0]["nid"]) == 128
    assert res[0]["rows"].tolist() == [0, 515] and res[1]["rows"].tolist() == [515, 1030]
    # identical summed norms and identical selection on both ranks
    assert np.array_equal(res[0]["norms"], res[1]["norms"])
    assert np.array_equal(res[0]["idx"], res[1]["idx"])
    # the exchange reproduces the unsharded norms and (up to R3 boundary swaps) selection
    n, m = 1030, 700
    G = synth.grad(n, m, layer=3, step=0, scale_exp=synth.col_scale_init(m, layer=3), dtype="fp32")
    whole = orc.column_norms(G)
    assert np.allclose(res[0]["norms"], whole, rtol=1e-6, atol=0)
    want = orc.topk(whole, orc.k_for(m, 100000))
    diff = set(res[0]["idx"].tolist()) ^ set(want.tolist())
    kth = np.min(whole[want])
    assert all(abs(whole[j] - kth) <= 1e-5 * kth for j in diff)


def test_shard_rows_product_helper():
    from paper_2505_12242_b200.dist import shard_rows
    assert [shard_rows(4096, 4, r) for r in range(4)] == [(0, 1024), (1024, 2048), (2048, 3072), (3072, 4096)]
    assert [shard_rows(5, 2, r) for r in range(2)] == [(0, 3), (3, 5)]
    for n in (1, 7, 50257):
        for w in (1, 2, 3, 8):
            spans = [shard_rows(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    with pytest.raises(ValueError):
        shard_rows(10, 2, 2)


def _peer_worker(rank, world, port):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2505_12242_b200.dist import open_peer_exchange

    class FakeCtx:
        """Stands in for zf.Context: a 64-byte handle per rank, and what peer_open receives."""
        opened = None

        def peer_handle(self):
            return bytes([rank]) * 64

        def peer_open(self, handles):
            self.opened = handles

    ctx = FakeCtx()
    open_peer_exchange(ctx)
    # every rank receives every rank's handle, in rank order (zf_peer_open maps handle q as rank q)
    assert ctx.opened == [bytes([q]) * 64 for q in range(world)], ctx.opened
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_open_peer_exchange_gathers_handles_in_rank_order(world):
    """f4 (iii) setup: dist.open_peer_exchange all-gathers the ranks' IPC handles over the
    process group in rank order before zf_peer_open (the mapping itself needs a GPU:
    tests/test_gpu_multirank.py)."""
    mp.spawn(_peer_worker, args=(world, _free_port()), nprocs=world, join=True)
