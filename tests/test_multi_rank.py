"""World-size-2 gloo tests of the multi-GPU host logic (CPU): node-block
ownership, the spectrum-ring all-gather/reassembly used by bench.py, and the
pair-range sharding covering every pair exactly once."""
import os
import socket

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


def _worker(rank, world, port, n_nodes, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2303_03279_b200.shard import allgather_ring, node_block, shard_plan
        S, L, nb = 3, 2, 4
        n0, n1, nloc = node_block(n_nodes, world, rank)
        local = torch.zeros((S, L, nb, nloc), dtype=torch.complex128)
        ids = torch.arange(n0, n1, dtype=torch.float64)
        for s in range(S):
            for l in range(L):
                for b in range(nb):
                    local[s, l, b, : n1 - n0] = ids + 1j * (1000 * s + 100 * l + 10 * b)
        full = torch.empty((S, L, nb, n_nodes), dtype=torch.complex128)
        allgather_ring(local, full, dist)
        want = torch.arange(n_nodes, dtype=torch.float64)
        ok = all(torch.equal(full[s, l, b], want + 1j * (1000 * s + 100 * l + 10 * b))
                 for s in range(S) for l in range(L) for b in range(nb))
        (rb, re_), (p0, p1) = shard_plan(n_nodes, world, rank)
        rng = torch.tensor([p0, p1, rb, re_], dtype=torch.int64)
        allr = [torch.zeros(4, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allr, rng)
        q.put((rank, ok, [r.tolist() for r in allr]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_nodes", [130, 1000])
def test_two_rank_ring_gather_and_pair_sharding(n_nodes):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_nodes, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    P = n_nodes * (n_nodes - 1) // 2
    for rank, ok, ranges in res:
        assert ok, f"rank {rank}: reassembled ring mismatch"
        assert ranges[0][0] == 0 and ranges[-1][1] == P
        for a, b in zip(ranges, ranges[1:]):
            assert a[1] == b[0] and a[3] == b[2]
