"""Multi-GPU sharding of the pair space.

Rank r owns node block r for K1 (spectra), the spectrum ring is all-gathered
(the path's one exchange step), and rank r computes the balanced pair-row
range of cs_row_tile_range; its outputs cover a contiguous global pair range.
"""
from __future__ import annotations

import torch

from .plan import row_tile_range


def node_block(n_nodes: int, world: int, rank: int):
    """(n0, n1, nloc): rank's node block and the padded per-rank block size."""
    nloc = (n_nodes + world - 1) // world
    return min(rank * nloc, n_nodes), min((rank + 1) * nloc, n_nodes), nloc


def assemble_ring(gathered: torch.Tensor, n_nodes: int) -> torch.Tensor:
    """[world, S, L, nb, nloc] gathered node blocks -> [S, L, nb, n_nodes] ring."""
    w, S, L, nb, nloc = gathered.shape
    return gathered.permute(1, 2, 3, 0, 4).reshape(S, L, nb, w * nloc)[..., :n_nodes]


def allgather_ring(local: torch.Tensor, full: torch.Tensor, dist, scratch: torch.Tensor | None = None):
    """All-gather node-block rings ``local`` [S, L, nb, nloc] of every rank into
    ``full`` [S, L, nb, N] (NCCL all_gather_into_tensor; list all_gather for gloo)."""
    ws = dist.get_world_size()
    if scratch is None:
        scratch = torch.empty((ws,) + tuple(local.shape), dtype=local.dtype, device=local.device)
    # complex rings travel as their real (re, im) views
    loc_r = torch.view_as_real(local) if local.is_complex() else local
    scr_r = torch.view_as_real(scratch) if scratch.is_complex() else scratch
    if dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(scr_r.reshape(-1), loc_r.contiguous().reshape(-1))
    else:  # gloo: host tensors (device rings are staged through host memory)
        parts = [torch.empty_like(loc_r, device="cpu") for _ in range(ws)]
        dist.all_gather(parts, loc_r.contiguous().cpu())
        for w in range(ws):
            scr_r[w].copy_(parts[w])
    full.copy_(assemble_ring(scratch, full.shape[-1]))
    return full


def shard_plan(n_nodes: int, world: int, rank: int):
    """((row_tile_begin, row_tile_end), (pair_begin, pair_end)) of this rank."""
    return row_tile_range(n_nodes, world, rank)
