"""Row sharding across GPUs (one process per GPU) — SURVEY.md §8(e).

Rows of G are independent (reference proj/src/factor.cpp:97-108 computes
them in independent chunks; SPEC.md:220 requires worker-count invariance), so
the units are split into contiguous row ranges with no collective on G. The
only exchange is the per-γ basis (landmarks, L, γ) broadcast from rank 0.
"""
from __future__ import annotations

from typing import Tuple

import numpy as np

__all__ = ["row_shard", "broadcast_basis", "compute_g_sharded"]

ROW_ALIGN = 256  # one CTA-pair tile (2 x 128-row UMMA M halves)


def row_shard(n: int, world_size: int, rank: int, align: int = ROW_ALIGN) -> Tuple[int, int]:
    """Contiguous [begin, end) of rank's rows; boundaries are multiples of `align`
    (so no 256-row pair tile straddles two GPUs) and the union over ranks is [0, n)."""
    if world_size < 1 or not (0 <= rank < world_size):
        raise ValueError("invalid rank / world size")
    if n < 0:
        raise ValueError("negative row count")
    per = -(-n // world_size)
    per = -(-per // align) * align
    begin = min(n, rank * per)
    end = min(n, (rank + 1) * per)
    return begin, end


def broadcast_basis(landmarks: np.ndarray | None, L: np.ndarray | None, gamma: float | None,
                    group=None, device=None):
    """Broadcast the factor basis from rank 0 with torch.distributed.

    Rank 0 passes the arrays; other ranks pass None and receive them. Works with
    gloo (CPU tensors) and NCCL (CUDA tensors; pass device). Returns
    (landmarks, L, gamma) as numpy fp64 on every rank.
    """
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    dev = torch.device(device) if device is not None else torch.device("cpu")
    if rank == 0:
        lm = torch.as_tensor(np.ascontiguousarray(landmarks, np.float64), device=dev)
        Lt = torch.as_tensor(np.ascontiguousarray(L, np.float64), device=dev)
        meta = torch.tensor([lm.shape[0], lm.shape[1], Lt.shape[1], float(gamma)], dtype=torch.float64,
                            device=dev)
    else:
        meta = torch.zeros(4, dtype=torch.float64, device=dev)
    dist.broadcast(meta, src=0, group=group)
    B, d, b_eff, g = int(meta[0]), int(meta[1]), int(meta[2]), float(meta[3])
    if rank != 0:
        lm = torch.empty((B, d), dtype=torch.float64, device=dev)
        Lt = torch.empty((B, b_eff), dtype=torch.float64, device=dev)
    dist.broadcast(lm, src=0, group=group)
    dist.broadcast(Lt, src=0, group=group)
    return lm.cpu().numpy(), Lt.cpu().numpy(), g


def compute_g_sharded(ctx, X: np.ndarray, landmarks: np.ndarray | None, L: np.ndarray | None,
                      gamma: float | None, group=None):
    """One process per GPU under torch.distributed (torchrun): rank 0's basis (landmarks,
    L, γ) is broadcast (the only exchange), then every rank computes the
    G rows of its contiguous row_shard of X through its own context (`ctx`, e.g.
    Context(device_ids=[local_rank])) — no collective on G. X holds all n rows (or at least
    this rank's shard at the same offsets); other ranks may pass None for the basis.
    Returns (begin, end, G_local)."""
    import torch.distributed as dist

    lm, Lb, g = broadcast_basis(landmarks, L, gamma, group=group)
    b, e = row_shard(X.shape[0], dist.get_world_size(group), dist.get_rank(group))
    ctx.set_basis_dense(lm, Lb, g)
    return b, e, ctx.compute_g_dense(np.ascontiguousarray(X[b:e], dtype=np.float64))
