"""f1: the all-gather fused into the GEMM epilogue (-m gpu).

comet_w4ax_gemm_allgather / comet_w4ax_linear_allgather write a rank's
N-shard of Y into columns [col0, col0 + N) of EVERY destination buffer.  On
one GPU the P ranks are simulated one after another with P local buffers
standing in for the peers' P2P-mapped copies (the kernel cannot tell: both
are device addresses written by the TMA engine / the decode epilogue).
Bars: after all P calls every buffer holds the same full output, each shard
bit-identical to the plain comet_w4ax_gemm / comet_w4ax_linear of that shard
(same kernel, same problem); columns outside a call's shard untouched.
"""
import numpy as np
import pytest
import torch

from paper_2410_12168_b200 import comet, synth, tp

pytestmark = pytest.mark.gpu


def to_dev(a):
    return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("M,N,K,P,group", [(300, 896, 1024, 3, 128), (16, 1024, 2048, 4, 2048),
                                            (1030, 1536, 1024, 2, 1024), (64, 640, 1024, 8, 128)])
def test_gemm_allgather_into_every_destination(M, N, K, P, group):
    p = synth.make_problem(M, N, K, n8=2, seed=M + P)
    X, perm = to_dev(p["X"]), to_dev(p["perm"])
    bits = comet.BlockBits(p["bits"])
    Xq8, Xq4, Sx = comet.comet_quantize_act(X, bits, perm)
    _, _, per = tp.shard_rows(N, P, 0)
    sentinel = torch.tensor(-7.0, dtype=torch.float16)
    bufs = [torch.full((M, P * per), -7.0, dtype=torch.float16, device="cuda") for _ in range(P)]
    ref = []
    for r in range(P):
        W = to_dev(tp.shard_weight(p["W"], P, r))
        Wq, Sw = comet.comet_pack_weight(W, perm, group if group != K else K)
        ws = comet.new_workspace(comet.comet_w4ax_gemm_workspace_bytes(M, per, K), X.device)
        ref.append(comet.comet_w4ax_gemm(Xq8, Xq4, Sx, bits, Wq, Sw, group, workspace=ws).clone())
        dests = [bufs[r]] + [bufs[i] for i in range(P) if i != r]
        comet.comet_w4ax_gemm_allgather(Xq8, Xq4, Sx, bits, Wq, Sw, dests, P * per, r * per, group, workspace=ws)
        torch.cuda.synchronize()
        if r == 0:  # columns of the shards not yet written still hold the sentinel
            for b in bufs:
                assert torch.all(b[:, per:] == sentinel)
    full = torch.cat(ref, dim=1)
    for b in bufs:
        assert torch.equal(b.view(torch.int16), full.view(torch.int16))


@pytest.mark.parametrize("M,K,P", [(1024, 4096, 2), (16, 4096, 4)])
def test_linear_allgather_matches_sharded_linear(M, K, P):
    N = 1280
    p = synth.make_problem(M, N, K, n8=3, seed=11 + M)
    X, perm = to_dev(p["X"]), to_dev(p["perm"])
    bits = comet.BlockBits(p["bits"])
    _, _, per = tp.shard_rows(N, P, 0)
    bufs = [torch.zeros((M, P * per), dtype=torch.float16, device="cuda") for _ in range(P)]
    ref = []
    for r in range(P):
        W = to_dev(tp.shard_weight(p["W"], P, r))
        Wq, Sw = comet.comet_pack_weight(W, perm, 128)
        scratch = comet.new_workspace(comet.comet_w4ax_linear_scratch_bytes(M, per, K, bits), X.device)
        ref.append(comet.comet_w4ax_linear(X, bits, Wq, Sw, perm=perm, scratch=scratch).clone())
        dests = [bufs[r]] + [bufs[i] for i in range(P) if i != r]
        comet.comet_w4ax_linear_allgather(X, bits, Wq, Sw, dests, P * per, r * per, perm=perm, scratch=scratch)
    torch.cuda.synchronize()
    full = torch.cat(ref, dim=1)
    for b in bufs:
        assert torch.equal(b.view(torch.int16), full.view(torch.int16))


def test_allgather_argument_checks():
    p = synth.make_problem(64, 256, 512, n8=1, seed=3)
    X, W = to_dev(p["X"]), to_dev(p["W"])
    bits = comet.BlockBits(p["bits"])
    Wq, Sw = comet.comet_pack_weight(W, None, 128)
    scratch = comet.new_workspace(comet.comet_w4ax_linear_scratch_bytes(64, 256, 512, bits), X.device)
    buf = torch.zeros((64, 512), dtype=torch.float16, device="cuda")
    with pytest.raises(comet.CometError):  # host X: the fused path writes device buffers only
        comet.comet_w4ax_linear_allgather(X.cpu().pin_memory(), bits, Wq, Sw, [buf], 512, 0, scratch=scratch)
    with pytest.raises(comet.CometError):  # shard past the row
        comet.comet_w4ax_linear_allgather(X, bits, Wq, Sw, [buf], 512, 384, scratch=scratch)
    with pytest.raises(comet.CometError):  # more than 8 destinations
        comet.comet_w4ax_linear_allgather(X, bits, Wq, Sw, [buf] * 9, 512, 0, scratch=scratch)
    with pytest.raises(comet.CometError):  # unaligned column offset
        comet.comet_w4ax_linear_allgather(X, bits, Wq, Sw, [buf], 512, 4, scratch=scratch)


def test_symmetric_memory_single_rank():
    """The symmetric-memory plumbing of tp.FusedAllGatherOutput on a 1-rank
    NCCL group (the P2P peers of a real run are the same device pointers)."""
    import os
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29561")
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        M, N, K = 512, 768, 1024
        p = synth.make_problem(M, N, K, n8=2, seed=5)
        X, W, perm = to_dev(p["X"]), to_dev(p["W"]), to_dev(p["perm"])
        bits = comet.BlockBits(p["bits"])
        Wq, Sw = comet.comet_pack_weight(W, perm, 128)
        scratch = comet.new_workspace(comet.comet_w4ax_linear_scratch_bytes(M, N, K, bits), X.device)
        ref = comet.comet_w4ax_linear(X, bits, Wq, Sw, perm=perm, scratch=scratch).clone()
        out = tp.FusedAllGatherOutput(M, N, X.device)
        tp.fused_linear_allgather(comet, X, bits, Wq, Sw, out, perm=perm, scratch=scratch)
        torch.cuda.synchronize()
        assert torch.equal(out.full(N).view(torch.int16), ref.view(torch.int16))
    finally:
        if own:
            dist.destroy_process_group()
