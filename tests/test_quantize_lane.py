"""GPU parity of the thread-per-item quantizer (csrc/quantize_lane.cuh, M >= 512)
against the oracle (-m gpu).

The kernel rotates each block's gather walk by a per-block amount derived
from the permutation and writes its output in place through shared memory,
so the cases that matter are: permutations of every shape (the FMPQ layout
of synth = outliers first, the rest in order; a uniformly random one; none),
block counts that make a warp straddle two staged rows (nb = 112, 86), a
stage ring that wraps many times, ragged M (padding rows of Sx), INT8 blocks
anywhere (scattered mask), both output forms (the packed INT4 plane of
comet_quantize_act and the e4m3 operand of comet_w4ax_linear) and bf16
activations.  Bars: planes and Sx bit-exact; the linear path's Y
bit-identical to the two-call path (whose planes are checked here).
"""
import importlib

import numpy as np
import pytest
import torch

import oracle
from paper_2410_12168_b200 import comet, synth

pytestmark = pytest.mark.gpu


def to_dev(a):
    return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()


def make(M, K, n8, kind, seed, mask="scattered"):
    p = synth.make_problem(M, 128, K, n8=n8, seed=seed, mask=mask)
    if kind == "none":
        p["perm"] = None
    elif kind == "random":
        p["perm"] = np.random.default_rng(seed).permutation(K).astype(np.int32)
    return p


@pytest.mark.parametrize("M,K,n8", [(512, 1024, 2), (1000, 4096, 3), (2053, 14336, 11), (777, 11008, 9),
                                     (600, 128, 1), (513, 32768, 20), (4096, 2048, 0)])
@pytest.mark.parametrize("kind", ["fmpq", "random", "none"])
def test_lane_quantizer_planes_bit_exact(M, K, n8, kind):
    p = make(M, K, n8, kind, seed=M + K)
    bits = comet.BlockBits(p["bits"])
    g8, g4, gs = comet.comet_quantize_act(to_dev(p["X"]), bits, to_dev(p["perm"]))
    torch.cuda.synchronize()
    o8, o4, os_ = oracle.quantize_act(p["X"], p["bits"], p["perm"])
    assert np.array_equal(g8.cpu().numpy().view(np.uint8), o8.view(np.uint8))
    assert np.array_equal(g4.cpu().numpy().view(np.uint8), o4.view(np.uint8))
    assert np.array_equal(gs.cpu().numpy().view(np.uint32), os_.view(np.uint32))


@pytest.mark.parametrize("M,K,n8", [(1024, 4096, 3), (515, 14336, 11)])
def test_lane_quantizer_bf16_bit_exact(M, K, n8):
    O = importlib.import_module("oracle.fmpq_aux")
    p = make(M, K, n8, "fmpq", seed=5 + M)
    b16 = (p["X"].astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    bits = comet.BlockBits(p["bits"])
    g8, g4, gs = comet.comet_quantize_act_bf16(to_dev(b16.view(np.int16)).view(torch.bfloat16), bits,
                                               to_dev(p["perm"]))
    torch.cuda.synchronize()
    o8, o4, os_ = O.quantize_act_bf16(b16, p["bits"], p["perm"])
    assert np.array_equal(g8.cpu().numpy(), o8) and np.array_equal(g4.cpu().numpy(), o4)
    assert np.array_equal(gs.cpu().numpy().view(np.uint32), os_.view(np.uint32))


@pytest.mark.parametrize("M,K,n8,kind", [(1024, 4096, 3, "fmpq"), (1030, 14336, 11, "random"),
                                          (700, 2048, 2, "none")])
def test_lane_quantizer_e4_linear_matches_two_call_path(M, K, n8, kind):
    """comet_w4ax_linear's fused e4m3 output (kE4 lane kernel) gives the same Y
    bit for bit as comet_quantize_act (packed planes, checked above) followed by
    comet_w4ax_gemm."""
    p = make(M, K, n8, kind, seed=3 * M + 1)
    N = 640
    W = to_dev((np.random.default_rng(M).standard_normal((N, K)) / np.sqrt(K)).astype(np.float16))
    X, perm = to_dev(p["X"]), to_dev(p["perm"])
    bits = comet.BlockBits(p["bits"])
    Wq, Sw = comet.comet_pack_weight(W, perm, 128)
    Xq8, Xq4, Sx = comet.comet_quantize_act(X, bits, perm)
    ws = comet.new_workspace(comet.comet_w4ax_gemm_workspace_bytes(M, N, K), X.device)
    ref = comet.comet_w4ax_gemm(Xq8, Xq4, Sx, bits, Wq, Sw, 128, workspace=ws)
    scratch = comet.new_workspace(comet.comet_w4ax_linear_scratch_bytes(M, N, K, bits), X.device)
    Y = comet.comet_w4ax_linear(X, bits, Wq, Sw, perm=perm, group=128, scratch=scratch)
    torch.cuda.synchronize()
    assert np.array_equal(Y.cpu().numpy().view(np.uint16), ref.cpu().numpy().view(np.uint16))


@pytest.mark.parametrize("seed", range(8))
def test_lane_quantizer_random_configs(seed):
    """Random shapes, masks and permutations (M >= 512, K up to 28672): planes
    and Sx bit-exact; the e4m3 linear path identical to the two-call path."""
    rng = np.random.default_rng(1000 + seed)
    nb = int(rng.choice([1, 3, 8, 31, 32, 33, 64, 86, 112, 150, 224]))
    K = 128 * nb
    M = int(rng.integers(512, 2600))
    n8 = int(rng.integers(0, max(1, nb // 3) + 1))
    mask = str(rng.choice(["prefix", "scattered"]))
    kind = str(rng.choice(["fmpq", "random", "none"]))
    p = make(M, K, n8, kind, seed=seed, mask=mask)
    bits = comet.BlockBits(p["bits"])
    X, perm = to_dev(p["X"]), to_dev(p["perm"])
    g8, g4, gs = comet.comet_quantize_act(X, bits, perm)
    torch.cuda.synchronize()
    o8, o4, os_ = oracle.quantize_act(p["X"], p["bits"], p["perm"])
    assert np.array_equal(g8.cpu().numpy().view(np.uint8), o8.view(np.uint8))
    assert np.array_equal(g4.cpu().numpy().view(np.uint8), o4.view(np.uint8))
    assert np.array_equal(gs.cpu().numpy().view(np.uint32), os_.view(np.uint32))
    if K <= 8192:
        N = 384
        W = to_dev((rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float16))
        Wq, Sw = comet.comet_pack_weight(W, perm, K)
        ws = comet.new_workspace(comet.comet_w4ax_gemm_workspace_bytes(M, N, K), X.device)
        ref = comet.comet_w4ax_gemm(g8, g4, gs, bits, Wq, Sw, K, workspace=ws)
        scratch = comet.new_workspace(comet.comet_w4ax_linear_scratch_bytes(M, N, K, bits), X.device)
        Y = comet.comet_w4ax_linear(X, bits, Wq, Sw, perm=perm, group=K, scratch=scratch)
        torch.cuda.synchronize()
        assert np.array_equal(Y.cpu().numpy().view(np.uint16), ref.cpu().numpy().view(np.uint16))
