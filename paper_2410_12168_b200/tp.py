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


# ------------------------------------------- overlap ----
def chunk_bounds(M: int, chunks: int):
    """[(m0, m1)] splitting M rows into `chunks` near-equal contiguous ranges."""
    chunks = max(1, min(chunks, M)) if M > 0 else 1
    edges = [M * i // chunks for i in range(chunks + 1)]
    return [(edges[i], edges[i + 1]) for i in range(chunks) if edges[i + 1] > edges[i]]


def pipelined_linear_allgather(gemm_rows, M: int, per: int, chunks: int, dtype, device, group=None):
    """GEMM + all-gather with the exchange of row chunk i overlapping the GEMM
    of chunk i + 1 (the "overlapped" column of SURVEY 8(e): serial
    GEMM + AG -> max(GEMM, AG) when the chunks pipeline).

    gemm_rows(m0, m1, out) writes rows [m0, m1) of this rank's Y shard into
    out ([m1 - m0, per], contiguous) on the current stream.  Each chunk's
    all_gather is issued asynchronously right after its GEMM (NCCL runs it on
    its own stream after the GEMM's event; gloo on a helper thread), so the
    next chunk's GEMM is enqueued while the previous chunk is in flight.
    Returns (y_chunks, bounds): y_chunks[i] is [P, m1 - m0, per] (rank-major)
    and lives in one flat buffer; chunked_to_full reassembles [M x N].
    """
    world = dist.get_world_size(group)
    bounds = chunk_bounds(M, chunks)
    y_local = torch.empty((M, per), dtype=dtype, device=device)
    flat = torch.empty(world * M * per, dtype=dtype, device=device)
    y_chunks, works = [], []
    for m0, m1 in bounds:
        mc = m1 - m0
        gemm_rows(m0, m1, y_local[m0:m1])
        dst = flat[world * m0 * per: world * m1 * per].view(world, mc, per)
        works.append(dist.all_gather_into_tensor(dst.view(world * mc, per), y_local[m0:m1], group=group,
                                                 async_op=True))
        y_chunks.append(dst)
    for w in works:
        w.wait()
    return y_chunks, bounds


def chunked_to_full(y_chunks, bounds, N: int) -> torch.Tensor:
    """[P x mc x per] rank-major chunks -> [M x N] (drops the padding)."""
    return torch.cat([gathered_to_full(yc, N) for yc in y_chunks], dim=0)


# ----------------------------------- row-parallel (K) ----
# The down projection pairs with the N-sharded gate_up: rank r already holds
# the intermediate activations' channel slice that gate_up produced, so the
# down GEMM is sharded on its reduction axis K instead -- no all-gather of
# the intermediate, one reduce-scatter of the output.  Shards are whole
# 128-channel FMPQ blocks, each rank quantizes its own slice (its blocks'
# per-(row, block) scales are the ones the unsharded quantizer would compute;
# the permutation and precision mask are per shard, channels never cross
# ranks), runs the local W4Ax GEMM to an fp16 partial, and the partials are
# summed in fp32 by the reduce-scatter over token rows.
def shard_k(K: int, world: int, rank: int, block: int = 128):
    """(k0, k1): rank's contiguous K range, whole blocks (may be empty)."""
    nb = K // block
    per = -(-nb // world)
    k0 = min(rank * per, nb) * block
    return k0, min((rank * per + per), nb) * block


def row_parallel_reduce(y_partial: torch.Tensor, group=None, scatter: bool = True) -> torch.Tensor:
    """Sum the ranks' [M x N] fp16 partials in fp32.  scatter: each rank gets
    its contiguous block of ceil(M / P) token rows (reduce-scatter; the last
    rank's block may be short), else the full sum on every rank (all-reduce).
    Returns fp32."""
    world = dist.get_world_size(group)
    M, N = y_partial.shape
    y32 = y_partial.to(torch.float32)
    if not scatter:
        dist.all_reduce(y32, group=group)
        return y32
    per = -(-M // world)
    buf = torch.zeros((per * world, N), dtype=torch.float32, device=y32.device)
    buf[:M] = y32
    out = torch.empty((per, N), dtype=torch.float32, device=y32.device)
    dist.reduce_scatter_tensor(out, buf, group=group)
    rank = dist.get_rank(group)
    return out[: max(0, min(per, M - rank * per))]


# ------------------------- all-gather fused into the GEMM ----
class FusedAllGatherOutput:
    """The full-width output [M x P*per] fp16 of an N-sharded layer in
    symmetric memory (torch.distributed._symmetric_memory: one allocation per
    rank, every peer's copy mapped into this process over NVLink P2P).  Each
    rank's comet_w4ax_linear_allgather writes its shard's Y tiles straight into
    ALL ranks' copies from the GEMM epilogue (the all-gather fused
    into the epilogue); barrier() is the single cross-rank sync after which
    every rank's copy holds the whole Y.  No NCCL call and no reassembly
    kernel on this path."""

    def __init__(self, M: int, per: int, device, group=None):
        import torch.distributed._symmetric_memory as symm_mem
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.per = per
        self.buf = symm_mem.empty((M, self.world * per), dtype=torch.float16, device=device)
        grp = group if group is not None else dist.group.WORLD
        self.handle = symm_mem.rendezvous(self.buf, grp)
        self.ptrs = [int(self.handle.buffer_ptrs[r]) for r in range(self.world)]

    def dests(self):
        """this rank's copy first, then the peers' (the C ABI's Ys[])"""
        return [self.ptrs[self.rank]] + [self.ptrs[r] for r in range(self.world) if r != self.rank]

    @property
    def ldy(self):
        return self.world * self.per

    @property
    def col0(self):
        return self.rank * self.per

    def barrier(self):
        self.handle.barrier()

    def full(self, N: int) -> torch.Tensor:
        return self.buf[:, :N]


def fused_linear_allgather(comet_mod, X, bits, Wq_shard, Sw_shard, out: FusedAllGatherOutput, perm=None,
                           group_size: int = 128, scratch=None, stream=None):
    """One N-sharded layer: quantize + GEMM whose epilogue stores into every
    rank's copy of `out`, then the one barrier."""
    comet_mod.comet_w4ax_linear_allgather(X, bits, Wq_shard, Sw_shard, out.dests(), out.ldy, out.col0, perm=perm,
                                          group=group_size, scratch=scratch, stream=stream)
    out.barrier()
