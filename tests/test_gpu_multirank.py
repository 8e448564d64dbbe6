"""The multi-GPU path on one GPU: node-block K1, the fp32 ring pushed into every
peer's ring (cs_ring_push), balanced row-tile shards, and the exact-sign fallback
reading remote nodes' fp64 spectra through the peer table.  The concatenated
shard outputs equal the single-plan run bit for bit (per-bin values; band means
within fp32 atomics-order noise of the fallback's band adds).

Ranks whose kernels wait on one another are never run on one GPU: each rank's
push completes (stream sync) before a host barrier, then the pair kernels run.
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch

from paper_2303_03279_b200.plan import SEVEN, DevicePlan, compute_connectivity, pow2_scale
from paper_2303_03279_b200.shard import RingExchange, node_block, shard_plan

pytestmark = pytest.mark.gpu


def _data(K=11, N=300, T=200, seed=9):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((K, N, T)).astype(np.float32)
    x[:, N - 5] = 0.7 * x[:, 3]          # zero-lag copy across node blocks: fp64 fallback reads remote X64
    x[:, 150] = 0.0                      # a dead node
    return x


def _single(x, nfft, lo, hi, taper, scale):
    xt = torch.tensor(x, device="cuda")
    plan = DevicePlan(x.shape[1], x.shape[2], nfft, lo, hi, taper=taper, slot_capacity=x.shape[0], device="cuda",
                      scale=scale)
    plan.spectra(xt, 0)
    return plan.pair_metrics(torch.arange(x.shape[0], dtype=torch.int32, device="cuda"), SEVEN + ("COHY",))


def _check(outs, full, world, N):
    for r, o in enumerate(outs):
        (_, _), (p0, p1) = shard_plan(N, world, r)
        for m in SEVEN + ("COHY",):
            assert torch.equal(o[m]["bins"].cuda(), full[m]["bins"][:, p0:p1]), (r, m)
            d = (o[m]["band"].cuda() - full[m]["band"][p0:p1]).abs().max()
            assert float(d) <= 1e-6, (r, m, float(d))


@pytest.mark.parametrize("world", [2, 3])
def test_ring_push_shards_reproduce_single_plan(world):
    K, N, T, nfft, lo, hi = 11, 300, 200, 256, 4, 30
    x = _data(K, N, T)
    scale = pow2_scale(float(np.abs(x).max()), min(T, nfft))
    full = _single(x, nfft, lo, hi, "hann", scale)
    plans = [DevicePlan(N, T, nfft, lo, hi, taper="hann", slot_capacity=K, device="cuda", scale=scale)
             for _ in range(world)]
    ex = RingExchange.local(plans)
    xt = torch.tensor(x, device="cuda")
    for e in ex:                        # K1 on each rank's block, then the exchange
        e.spectra(xt[:, e.n0:e.n1])
    for e in ex:
        e.push(0, K)
    torch.cuda.synchronize()
    slots = torch.arange(K, dtype=torch.int32, device="cuda")
    outs = []
    for r, e in enumerate(ex):
        (rb, re), (p0, p1) = shard_plan(N, world, r)
        outs.append(e.plan.pair_metrics(slots, SEVEN + ("COHY",), row_tiles=(rb, re), pair_base=p0,
                                        pair_count=p1 - p0))
    torch.cuda.synchronize()
    assert sum(p.guard_stats()["flagged"] for p in plans) > 0      # the fallback ran (remote X64 reads)
    _check(outs, full, world, N)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, path, args):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        K, N, T, nfft, lo, hi, scale = args
        x = _data(K, N, T)
        plan = DevicePlan(N, T, nfft, lo, hi, taper="hann", slot_capacity=K, device="cuda", scale=scale)
        ex = RingExchange(plan, dist)              # CUDA IPC handles over gloo
        n0, n1, _ = node_block(N, world, rank)
        ex.spectra(torch.tensor(x[:, n0:n1], device="cuda"))
        ex.push(0, K)
        torch.cuda.synchronize()
        dist.barrier()                             # every push into every ring is complete
        (rb, re), (p0, p1) = shard_plan(N, world, rank)
        o = plan.pair_metrics(torch.arange(K, dtype=torch.int32, device="cuda"), SEVEN + ("COHY",),
                              row_tiles=(rb, re), pair_base=p0, pair_count=p1 - p0)
        torch.cuda.synchronize()
        dist.barrier()                             # peers may still read our fp64 ring in their fallback
        torch.save({m: {k: v.cpu() for k, v in d.items()} for m, d in o.items()}, f"{path}/rank{rank}.pt")
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_two_processes_ipc_rings_reproduce_single_plan():
    """bench.py's N > 1 path in two processes sharing one GPU (gloo for the host
    handshakes, CUDA IPC for the rings)."""
    import torch.multiprocessing as mp
    K, N, T, nfft, lo, hi = 11, 300, 200, 256, 4, 30
    x = _data(K, N, T)
    scale = pow2_scale(float(np.abs(x).max()), min(T, nfft))
    full = _single(x, nfft, lo, hi, "hann", scale)
    world = 2
    with tempfile.TemporaryDirectory() as d:
        ctx = mp.get_context("spawn")
        port = _free_port()
        procs = [ctx.Process(target=_rank_main, args=(r, world, port, d, (K, N, T, nfft, lo, hi, scale)))
                 for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(timeout=300)
            assert p.exitcode == 0
        outs = [torch.load(f"{d}/rank{r}.pt") for r in range(world)]
    _check(outs, full, world, N)
