"""N>1 path on CPU: world_size-2 gloo run of the N-sharded W4Ax layer
(-m "not gpu").  The per-rank GEMM is the oracle here (no GPU); the sharding,
the all_gather and the reassembly are the product code (tp.py) that bench.py
runs over NCCL on GPUs.  The gathered Y must equal the single-process Y
bit for bit (each output channel depends only on its own weight row)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2410_12168_b200 import synth, tp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, M, N, K, group, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = synth.make_problem(M, N, K, n8=1, seed=31)
        Wl = tp.shard_weight(p["W"], world, rank)
        g = K if group == "K" else 128
        Xq8, Xq4, Sx = oracle.quantize_act(p["X"], p["bits"], p["perm"])
        Wq, Sw = oracle.pack_weight(Wl, g, p["perm"])
        y = oracle.w4ax_gemm(Xq8, Xq4, Sx, p["bits"], Wq, Sw, group=g)["y"]
        # gloo has no fp16/int16 transport: carry the fp16 values in fp32 (exact)
        y_all = tp.all_gather_y(torch.from_numpy(y.astype(np.float32)))
        full = tp.gathered_to_full(y_all, N).numpy().astype(np.float16)
        # every rank's activation planes are identical (replicated X)
        digest = torch.tensor([int(Xq4.astype(np.int64).sum()), int(Xq8.astype(np.int64).sum())])
        allx = [torch.zeros_like(digest) for _ in range(world)]
        dist.all_gather(allx, digest)
        q.put((rank, full, [t.tolist() for t in allx]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("N,group", [(640, 128), (512, "K"), (1152, 128)])
def test_n_sharded_allgather_equals_single_process(N, group):
    M, K, world = 12, 512, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, M, N, K, group, q)) for r in range(world)]
    for p_ in procs:
        p_.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    p = synth.make_problem(M, N, K, n8=1, seed=31)
    g = K if group == "K" else 128
    Xq8, Xq4, Sx = oracle.quantize_act(p["X"], p["bits"], p["perm"])
    Wq, Sw = oracle.pack_weight(p["W"], g, p["perm"])
    ref = oracle.w4ax_gemm(Xq8, Xq4, Sx, p["bits"], Wq, Sw, group=g)["y"]
    for rank, full, digests in res:
        assert np.array_equal(full.view(np.uint16), ref.view(np.uint16)), rank
        assert all(d == digests[0] for d in digests)


def test_shard_rows_cover_and_align():
    for N in (4096, 11008, 57344, 8192, 10240, 640):
        for world in (1, 2, 4, 8):
            seen = []
            for r in range(world):
                n0, n1, per = tp.shard_rows(N, world, r)
                assert per % 128 == 0 and n1 - n0 <= per
                seen.extend(range(n0, n1))
            assert seen == list(range(N))


def test_gathered_to_full_layout():
    y_all = torch.arange(2 * 3 * 4).reshape(2, 3, 4)
    full = tp.gathered_to_full(y_all, 7)
    assert full.tolist() == [[0, 1, 2, 3, 12, 13, 14], [4, 5, 6, 7, 16, 17, 18], [8, 9, 10, 11, 20, 21, 22]]


def _worker_pipelined(rank, world, port, M, N, K, chunks, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = synth.make_problem(M, N, K, n8=1, seed=37)
        Wl = tp.shard_weight(p["W"], world, rank)
        n0, n1, per = tp.shard_rows(N, world, rank)
        Xq8, Xq4, Sx = oracle.quantize_act(p["X"], p["bits"], p["perm"])
        Wq, Sw = oracle.pack_weight(Wl, 128, p["perm"])
        y = oracle.w4ax_gemm(Xq8, Xq4, Sx, p["bits"], Wq, Sw, group=128)["y"]
        calls = []

        def gemm_rows(m0, m1, out):  # stand-in for the device GEMM of rows [m0, m1)
            calls.append((m0, m1))
            out.copy_(torch.from_numpy(y[m0:m1].astype(np.float32)))

        yc, bounds = tp.pipelined_linear_allgather(gemm_rows, M, per, chunks, torch.float32, "cpu")
        full = tp.chunked_to_full(yc, bounds, N).numpy().astype(np.float16)
        q.put((rank, full, calls))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("chunks", [1, 3, 4])
def test_pipelined_gemm_allgather_equals_single_process(chunks):
    """f1: the chunked GEMM/all-gather pipeline reassembles the same Y."""
    M, N, K, world = 10, 640, 256, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_pipelined, args=(r, world, port, M, N, K, chunks, q)) for r in range(world)]
    for p_ in procs:
        p_.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    p = synth.make_problem(M, N, K, n8=1, seed=37)
    Xq8, Xq4, Sx = oracle.quantize_act(p["X"], p["bits"], p["perm"])
    Wq, Sw = oracle.pack_weight(p["W"], 128, p["perm"])
    ref = oracle.w4ax_gemm(Xq8, Xq4, Sx, p["bits"], Wq, Sw, group=128)["y"]
    for rank, full, calls in res:
        assert np.array_equal(full.view(np.uint16), ref.view(np.uint16)), rank
        assert calls == tp.chunk_bounds(M, chunks)


def test_chunk_bounds():
    assert tp.chunk_bounds(10, 3) == [(0, 3), (3, 6), (6, 10)]
    assert tp.chunk_bounds(2, 4) == [(0, 1), (1, 2)]
    assert tp.chunk_bounds(7, 1) == [(0, 7)]


# ------------------------------------------ f4: row-parallel (K-sharded) ----
def _k_partial(p, k0, k1):
    """oracle partial of one K shard: the shard's blocks quantized on their own
    (identity permutation inside the shard), fp16 Y."""
    if k1 <= k0:
        return np.zeros((p["X"].shape[0], p["W"].shape[0]), np.float16)
    bits = p["bits"][k0 // 128:k1 // 128]
    Xs = np.ascontiguousarray(p["X"][:, k0:k1])
    Ws = np.ascontiguousarray(p["W"][:, k0:k1])
    Xq8, Xq4, Sx = oracle.quantize_act(Xs, bits)
    Wq, Sw = oracle.pack_weight(Ws, 128)
    return oracle.w4ax_gemm(Xq8, Xq4, Sx, bits, Wq, Sw, group=128)["y"]


def _worker_rowpar(rank, world, port, M, N, K, scatter, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = synth.make_problem(M, N, K, n8=2, seed=41)
        k0, k1 = tp.shard_k(K, world, rank)
        y = _k_partial(p, k0, k1)
        out = tp.row_parallel_reduce(torch.from_numpy(y.astype(np.float32)).half(), scatter=scatter)
        q.put((rank, out.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("M,K,world,scatter", [(12, 512, 2, True), (13, 640, 2, True), (12, 512, 2, False)])
def test_row_parallel_k_sharded_equals_sum_of_shards(M, K, world, scatter):
    N = 256
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_rowpar, args=(r, world, port, M, N, K, scatter, q)) for r in range(world)]
    for p_ in procs:
        p_.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    p = synth.make_problem(M, N, K, n8=2, seed=41)
    parts = [_k_partial(p, *tp.shard_k(K, world, r)).astype(np.float32) for r in range(world)]
    total = parts[0] + parts[1]  # fp32, the order gloo/NCCL use for two ranks is immaterial (commutative)
    per = -(-M // world)
    for r in range(world):
        want = total[r * per:min(M, (r + 1) * per)] if scatter else total
        assert np.array_equal(res[r], want), r
    # against the unsharded path: whole 128-blocks keep every (row, block)
    # scale and INT32 block sum; only the fp16 rounding of each partial and
    # the block-to-shard assignment of the INT8 blocks' planes differ
    Xq8, Xq4, Sx = oracle.quantize_act(p["X"], p["bits"])
    Wq, Sw = oracle.pack_weight(p["W"], 128)
    ref = oracle.w4ax_gemm(Xq8, Xq4, Sx, p["bits"], Wq, Sw, group=128, want_y64=True)["y64"]
    bound = world * 2.0 ** -11 * np.max(np.abs(np.stack(parts)), axis=0) + 1e-6
    assert np.all(np.abs(total - ref) <= bound + 2.0 ** -11 * np.abs(ref))


def test_shard_k_blocks_cover():
    for K, world in [(512, 2), (640, 4), (28672, 8), (128, 2)]:
        rs = [tp.shard_k(K, world, r) for r in range(world)]
        assert rs[0][0] == 0 and max(r[1] for r in rs) == K
        for (a0, a1), (b0, b1) in zip(rs, rs[1:]):
            assert a1 == b0 or (b0 == b1 == K)
        assert all(k0 % 128 == 0 and k1 % 128 == 0 for k0, k1 in rs)


@pytest.mark.gpu
def test_row_parallel_shards_through_the_cuda_path():
    """The two K shards' local GEMMs run through the C ABI (one GPU, shards in
    sequence) and their fp32 sum matches the oracle's shard sum within the
    per-partial Y tolerance."""
    from paper_2410_12168_b200 import comet

    M, N, K, world = 300, 512, 1024, 2
    p = synth.make_problem(M, N, K, n8=2, seed=43)
    dev = torch.device("cuda")
    total = np.zeros((M, N), np.float64)
    bound = np.zeros((M, N), np.float64)
    gpu = np.zeros((M, N), np.float32)
    for r in range(world):
        k0, k1 = tp.shard_k(K, world, r)
        bits = p["bits"][k0 // 128:k1 // 128]
        Xs = torch.from_numpy(np.ascontiguousarray(p["X"][:, k0:k1])).to(dev)
        Ws = torch.from_numpy(np.ascontiguousarray(p["W"][:, k0:k1])).to(dev)
        Xq8, Xq4, Sx = comet.comet_quantize_act(Xs, bits)
        Wq, Sw = comet.comet_pack_weight(Ws, None, 128)
        ws = comet.new_workspace(comet.comet_w4ax_gemm_workspace_bytes(M, N, k1 - k0), dev)
        y = comet.comet_w4ax_gemm(Xq8, Xq4, Sx, bits, Wq, Sw, 128, workspace=ws)
        gpu += y.float().cpu().numpy()
        ref = _k_partial(p, k0, k1).astype(np.float64)
        total += ref
        bound += np.maximum(2.0 ** -10 * np.abs(ref), 1e-3)
    assert np.all(np.abs(gpu - total) <= bound)


def test_fused_allgather_destination_order():
    """f1 host logic: this rank's copy first, then the peers' (the C ABI's
    Ys[]), the shard's column offset and the full row stride."""
    o = tp.FusedAllGatherOutput.__new__(tp.FusedAllGatherOutput)
    o.world, o.rank, o.per = 4, 2, 384
    o.ptrs = [1000, 2000, 3000, 4000]
    assert o.dests() == [3000, 1000, 2000, 4000]
    assert o.col0 == 768 and o.ldy == 1536
