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


def all_gather_outputs(packed, group=None):
    """All-gather equally sized per-rank blocks (torch tensors) -> (world*P, 14)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    out = torch.empty((world * packed.shape[0], packed.shape[1]), dtype=packed.dtype, device=packed.device)
    dist.all_gather_into_tensor(out, packed.contiguous(), group=group)
    return out
