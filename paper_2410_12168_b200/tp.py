"""N-sharded tensor parallelism for the W4Ax linear layer (BJ north_star).

Rank r of P owns output channels [n0, n1) = shard_rows(N, P, r): a contiguous
range padded to a multiple of 128 so every shard is a valid comet_w4ax_gemm
problem (N % 128 == 0).  X, perm and block_bits are replicated; every rank
quantizes the same X (bit-identical planes), runs its local GEMM, and the only
exchange step is one all_gather of the Y shards (NCCL over NVLink/NVSwitch on
GPUs, gloo in the CPU tests).  Each output column depends only on its weight
row, so no other communication is needed.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def shard_rows(N: int, world: int, rank: int, align: int = 128):
    """(n0, n1, width): rank's channel range and the padded shard width."""
    per = -(-N // world)
    per = -(-per // align) * align
    n0 = min(rank * per, N)
    return n0, min(n0 + per, N), per


def shard_weight(W: np.ndarray, world: int, rank: int, align: int = 128) -> np.ndarray:
    """Rank's rows of W [N x K], zero-padded to the shard width."""
    N, K = W.shape
    n0, n1, per = shard_rows(N, world, rank, align)
    out = np.zeros((per, K), W.dtype)
    out[: n1 - n0] = W[n0:n1]
    return out


def all_gather_y(y_local: torch.Tensor, out: torch.Tensor | None = None, group=None) -> torch.Tensor:
    """Gather [M x width] shards from every rank into [P x M x width] (rank-major)."""
    world = dist.get_world_size(group)
    M, per = y_local.shape
    if out is None:
        out = torch.empty((world, M, per), dtype=y_local.dtype, device=y_local.device)
    # flat [P*M x width] view: accepted by both NCCL and gloo
    dist.all_gather_into_tensor(out.view(world * M, per), y_local.contiguous(), group=group)
    return out


def gathered_to_full(y_all: torch.Tensor, N: int) -> torch.Tensor:
    """[P x M x width] rank-major shards -> [M x N] (drops the padding)."""
    P, M, per = y_all.shape
    return y_all.permute(1, 0, 2).reshape(M, P * per)[:, :N]
