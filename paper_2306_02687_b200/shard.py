"""Macro Gauss points across ranks (one process per GPU).

The points are independent ("parallelize over macro
integration points"), so every rank owns a contiguous block and evaluates it
with its own engine; per-point input streams are keyed by the global point
index (fe2_paths p0), so a shard computes bit for bit what a single GPU
computes for the same points. The only exchange is the one the monolithic
scheme needs after every increment: the macro stress, condensed tangent,
residual norm and status of every point, all-gathered (NCCL on GPUs, gloo in
the CPU tests).
"""
from __future__ import annotations

import numpy as np

PACK = 14  # sigma(3) + C(9) + res(1) + status(1), fp64


def shard_range(P_total: int, rank: int, world: int) -> tuple[int, int]:
    """[p0, p1) of rank's contiguous, balanced block."""
    base, rem = divmod(P_total, world)
    p0 = rank * base + min(rank, rem)
    return p0, p0 + base + (1 if rank < rem else 0)


def gather_rows(counts, P_max=None):
    """Row indices of the real points in a gathered buffer of world blocks of
    P_max rows (fe2_hrom_gather's layout: rank r's points first in block r, the
    rest of the block is padding with status -1). counts = points per rank."""
    P_max = max(counts) if P_max is None else P_max
    return np.concatenate([np.arange(r * P_max, r * P_max + c) for r, c in enumerate(counts)])


def pad_block(packed, P_max):
    """This rank's packed records padded to P_max rows the way the device packs
    them (NaN values, status -1), numpy or torch."""
    P = packed.shape[0]
    if isinstance(packed, np.ndarray):
        out = np.full((P_max, packed.shape[1]), np.nan)
        out[:, -1] = -1.0
    else:
        import torch

        out = torch.full((P_max, packed.shape[1]), float("nan"), dtype=packed.dtype, device=packed.device)
        out[:, -1] = -1.0
    out[:P] = packed
    return out


def pack_outputs(sigma, C, res, status):
    """(P,3), (P,3,3)|(P,9), (P,), (P,) -> (P,14) float64 (numpy or torch)."""
    P = sigma.shape[0]
    if isinstance(sigma, np.ndarray):
        out = np.empty((P, PACK))
        out[:, 0:3] = sigma
        out[:, 3:12] = C.reshape(P, 9)
        out[:, 12] = res
        out[:, 13] = status
        return out
    import torch

    out = torch.empty((P, PACK), dtype=torch.float64, device=sigma.device)
    out[:, 0:3] = sigma
    out[:, 3:12] = C.reshape(P, 9)
    out[:, 12] = res
    out[:, 13] = status.to(torch.float64)
    return out


def unpack_outputs(packed):
    P = packed.shape[0]
    return dict(sigma=packed[:, 0:3], C=packed[:, 3:12].reshape(P, 3, 3), res_norm=packed[:, 12],
                status=packed[:, 13].astype(np.int32) if isinstance(packed, np.ndarray) else packed[:, 13].int())


def all_gather_counts(P_local, group=None):
    """Every rank's point count (the layout fe2_hrom_gather_layout exchanges)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    out = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(out, torch.tensor([P_local], dtype=torch.int64), group=group)
    return [int(t.item()) for t in out]


def all_gather_outputs(packed, group=None):
    """All-gather equally sized per-rank blocks (torch tensors) -> (world*P, 14)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    out = torch.empty((world * packed.shape[0], packed.shape[1]), dtype=packed.dtype, device=packed.device)
    dist.all_gather_into_tensor(out, packed.contiguous(), group=group)
    return out
