"""Multi-GPU sharding of the pair space.

One process per GPU, each holding a plan over all N nodes.  Rank r computes K1
for its node block only, pushes that block of its fp32 spectrum ring into every
peer's ring over NVLink peer memory (``RingExchange.push``: strided copy-engine
copies through IPC-mapped peer rings, csconn ``cs_ring_push``), and after one
barrier computes the balanced pair-row range of ``cs_row_tile_range``; its
outputs cover a contiguous global pair range and stay on the rank.  The fp64 ring
is never exchanged: the rare exact-sign fallback reads remote nodes' fp64
spectra from the owning rank's ring (P2P loads through the attached pointer
table).  The reference has no multi-process path.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from .plan import _stream_ptr, row_tile_range


def node_block(n_nodes: int, world: int, rank: int):
    """(n0, n1, nloc): rank's node block and the per-rank block size (node n is
    owned by rank n // nloc)."""
    nloc = (n_nodes + world - 1) // world
    return min(rank * nloc, n_nodes), min((rank + 1) * nloc, n_nodes), nloc


def shard_plan(n_nodes: int, world: int, rank: int):
    """((row_tile_begin, row_tile_end), (pair_begin, pair_end)) of this rank."""
    return row_tile_range(n_nodes, world, rank)


def exchange_handles(dist, mine: bytes) -> list:
    """Every rank's ring handle bytes, in rank order (host objects over ``dist``)."""
    allh = [None] * dist.get_world_size()
    dist.all_gather_object(allh, mine)
    if any(len(h) != len(mine) for h in allh):
        raise RuntimeError("ring handles of different sizes: mismatched csconn builds across ranks")
    return allh


class RingExchange:
    """The ring exchange of one rank's plan with its peers.

    ``RingExchange(plan, dist)`` exports this rank's ring (CUDA IPC handles),
    all-gathers the handles over ``dist`` (any backend: they are host bytes) and
    maps every peer's ring; ``RingExchange.local(plans)`` wires plans living in
    one process (tests) by device pointers instead."""

    def __init__(self, plan, dist=None, world: int | None = None, rank: int | None = None, _ptrs=None):
        self.plan = plan
        self.world = dist.get_world_size() if dist is not None else int(world)
        self.rank = dist.get_rank() if dist is not None else int(rank)
        self.n0, self.n1, self.nloc = node_block(plan.n_nodes, self.world, self.rank)
        L = _lib.lib()
        if _ptrs is not None:
            x64, x32 = _ptrs
            a64 = (ctypes.c_void_p * self.world)(*x64)
            a32 = (ctypes.c_void_p * self.world)(*x32)
            _lib.check(L.cs_ring_attach_ptrs(plan._h, a64, a32, self.world, self.rank, self.nloc))
            return
        h = _lib.CsRingHandle()
        _lib.check(L.cs_ring_export(plan._h, ctypes.byref(h)))
        allh = exchange_handles(dist, bytes(bytearray(h)))
        arr = (_lib.CsRingHandle * self.world)()
        for r, raw in enumerate(allh):
            ctypes.memmove(ctypes.byref(arr[r]), raw, ctypes.sizeof(_lib.CsRingHandle))
        _lib.check(L.cs_ring_attach(plan._h, arr, self.world, self.rank, self.nloc))

    @classmethod
    def local(cls, plans):
        """Exchanges among plans of this process (one per simulated rank)."""
        x64, x32 = [], []
        for p in plans:
            a, b, n = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int64()
            _lib.check(_lib.lib().cs_ring_view(p._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(n)))
            x64.append(a.value)
            x32.append(b.value)
        return [cls(p, world=len(plans), rank=r, _ptrs=(x64, x32)) for r, p in enumerate(plans)]

    def spectra(self, x_block: torch.Tensor, slot0: int = 0, stream=None) -> None:
        """K1 for this rank's node block; x_block [k, n1 - n0, T] on the plan's device."""
        self.plan.spectra_nodes(x_block, self.n0, slot0, stream=stream)

    def push(self, slot0: int, k_count: int, stream=None) -> None:
        """This rank's block of slots slot0 .. slot0 + k_count - 1 into every peer's ring."""
        _lib.check(_lib.lib().cs_ring_push(self.plan._h, self.n0, self.n1 - self.n0, int(slot0), int(k_count),
                                           _stream_ptr(stream)))
