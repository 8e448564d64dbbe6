"""World-size-2 gloo tests of the multi-GPU host logic (CPU): node-block
ownership (node n lives on rank n // nloc, the table the fp64 fallback reads
through), the ring-handle exchange used by shard.RingExchange, and the
pair-range sharding covering every pair exactly once."""
import os
import socket

import pytest
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
        from paper_2303_03279_b200.shard import exchange_handles, node_block, shard_plan
        n0, n1, nloc = node_block(n_nodes, world, rank)
        owner_ok = all(n // nloc == rank for n in range(n0, n1))
        # handle bytes of the size of a csconn ring handle (2 x 64 B IPC + geometry)
        mine = bytes([rank]) * 144
        allh = exchange_handles(dist, mine)
        ex_ok = [h[0] for h in allh] == list(range(world))
        (rb, re_), (p0, p1) = shard_plan(n_nodes, world, rank)
        q.put((rank, owner_ok and ex_ok, (n0, n1), (p0, p1, rb, re_)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_nodes", [130, 1000, 10242])
def test_two_rank_blocks_handles_and_pair_sharding(n_nodes):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_nodes, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    P = n_nodes * (n_nodes - 1) // 2
    assert all(ok for _, ok, _, _ in res)
    blocks = [b for _, _, b, _ in res]
    assert blocks[0][0] == 0 and blocks[-1][1] == n_nodes
    assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
    ranges = [r for _, _, _, r in res]
    assert ranges[0][0] == 0 and ranges[-1][1] == P
    for a, b in zip(ranges, ranges[1:]):
        assert a[1] == b[0] and a[3] == b[2]
