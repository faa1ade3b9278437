"""f4 FP16 weight-scale storage ("each group has one FP16 scale
factor"): comet_pack_weight_f16s / comet_w4ax_gemm_f16s.

-m "not gpu": the oracle (oracle.fmpq_aux.pack_weight_f16s) against the O5
oracle and the definition's closed-form properties.
-m gpu: packed weights and fp16 scales bit-exact, the GEMM within the Y
tolerance of the oracle on the fp32 values of the fp16 scales, and
bit-identical to comet_w4ax_gemm fed those fp32 scales.
"""
import numpy as np
import pytest

import oracle
from oracle import fmpq_aux as O
from paper_2410_12168_b200 import synth


def _unpack(Wq):
    lo = (Wq & 0xF).astype(np.int8)
    hi = (Wq >> 4).astype(np.int8)
    lo[lo > 7] -= 16
    hi[hi > 7] -= 16
    N, h = Wq.shape
    q = np.zeros((N, 2 * h), np.int8)
    # O4: per 8 values one LE word, byte j = e_j | e_{j+4} << 4
    for w in range(h // 4):
        for j in range(4):
            q[:, 8 * w + j] = lo[:, 4 * w + j]
            q[:, 8 * w + 4 + j] = hi[:, 4 * w + j]
    return q


@pytest.mark.parametrize("group", [128, 512])
def test_f16_scales_are_the_fp16_rounding_of_the_o5_scales(group):
    rng = np.random.default_rng(3)
    W = (rng.standard_normal((16, 512)) * 0.05).astype(np.float16)
    W[3, :group] = 0  # an all-zero group -> scale 1, codes 0
    _, Sw32 = oracle.pack_weight(W, group)
    Wq, Sw16 = O.pack_weight_f16s(W, group)
    assert np.array_equal(Sw16.view(np.uint16), Sw32.astype(np.float16).view(np.uint16))
    assert Sw16[0, 3] == 1.0 and not _unpack(Wq)[3, :group].any()


def test_exact_scales_give_the_o5_codes():
    # a = 7 * 2^k: a / 7 = 2^k is exact in fp16, w / s = w * (7 / a) exactly -> the O5 codes
    rng = np.random.default_rng(4)
    W = (rng.integers(-56, 57, size=(8, 256)) / 8.0).astype(np.float16)  # multiples of 1/8 in [-7, 7]
    W[:, 0] = 7.0
    W[:, 128] = -7.0
    Wq32, Sw32 = oracle.pack_weight(W, 128)
    Wq16, Sw16 = O.pack_weight_f16s(W, 128)
    assert np.array_equal(Sw16.astype(np.float32), Sw32) and np.array_equal(Wq16, Wq32)


def test_round_trip_bound_with_the_clamp():
    # |w - s q| <= s / 2 unless the fp16 rounding made s < a / 7 and the clamp fired,
    # where the error is |w| - 7 s <= a (1 - 7 s / a) <= a 2^-11 (one fp16 rounding)
    rng = np.random.default_rng(5)
    W = (rng.standard_normal((32, 256)) * np.exp(rng.uniform(-6, 3, size=(32, 1)))).astype(np.float16)
    Wq, Sw16 = O.pack_weight_f16s(W, 128)
    q = _unpack(Wq).astype(np.float64)
    s = np.repeat(Sw16.astype(np.float64).T, 128, axis=1)
    w = W.astype(np.float64)
    a = np.repeat(np.abs(w).reshape(32, 2, 128).max(axis=2), 128, axis=1)
    err = np.abs(w - s * q)
    assert np.all(err <= np.maximum(s / 2, a * 2.0 ** -11) * (1 + 2.0 ** -20) + 1e-30)
    assert np.all(np.abs(q) <= 7)


@pytest.mark.gpu
@pytest.mark.parametrize("M,N,K,group", [(16, 256, 512, 128), (300, 640, 1024, 128), (300, 640, 1024, 1024)])
def test_f16_scales_gpu_parity(M, N, K, group):
    import torch
    from paper_2410_12168_b200 import comet
    p = synth.make_problem(M, N, K, n8=2, seed=7 + M, mask="scattered")
    dev = torch.device("cuda")
    X, W, perm = (torch.from_numpy(p[k]).to(dev) for k in ("X", "W", "perm"))
    bits = comet.BlockBits(p["bits"])
    Wq, Sw16 = comet.comet_pack_weight_f16s(W, perm, group)
    oWq, oSw16 = O.pack_weight_f16s(p["W"], group, p["perm"])
    assert np.array_equal(comet.wq_tiled_to_rowmajor(Wq.cpu().numpy(), N, K), oWq)
    assert np.array_equal(Sw16.cpu().numpy().view(np.uint16), oSw16.view(np.uint16))
    Xq8, Xq4, Sx = comet.comet_quantize_act(X, bits, perm)
    Y = comet.comet_w4ax_gemm_f16s(Xq8, Xq4, Sx, bits, Wq, Sw16, group)
    ws = comet.new_workspace(comet.comet_w4ax_gemm_workspace_bytes(M, N, K), dev)
    Y32 = comet.comet_w4ax_gemm(Xq8, Xq4, Sx, bits, Wq, Sw16.float().contiguous(), group, workspace=ws)
    torch.cuda.synchronize()
    assert np.array_equal(Y.cpu().numpy().view(np.uint16), Y32.cpu().numpy().view(np.uint16))
    o8, o4, os_ = oracle.quantize_act(p["X"], p["bits"], p["perm"])
    ref = oracle.w4ax_gemm(o8, o4, os_, p["bits"], oWq, oSw16.astype(np.float32), group=group)["y"].astype(np.float64)
    y = Y.float().cpu().numpy().astype(np.float64)
    assert np.all(np.abs(y - ref) <= np.maximum(2.0 ** -10 * np.abs(ref), 1e-3))


# ---- BF16 scale storage (the other half of f4's "FP16/BF16") ----------------
def test_bf16_rounding_helper_matches_torch_rne():
    import torch
    rng = np.random.default_rng(9)
    x = np.concatenate([rng.standard_normal(4000).astype(np.float32) * np.float32(10.0) ** rng.integers(-30, 30, 4000),
                        np.array([1.0, 1 + 2 ** -8, 1 + 3 * 2 ** -8, 1 + 2 ** -8 + 2 ** -20, 3.0e38, 1e-38],
                                 np.float32)]).astype(np.float32)
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(O.f32_to_bf16_bits(x), ref)
    assert O.f32_to_bf16_bits(np.float32(1 + 2 ** -8)) == 0x3F80  # tie -> even
    assert O.f32_to_bf16_bits(np.float32(1 + 3 * 2 ** -8)) == 0x3F82


@pytest.mark.parametrize("group", [128, 512])
def test_bf16_scales_are_the_bf16_rounding_of_the_o5_scales(group):
    rng = np.random.default_rng(13)
    W = (rng.standard_normal((16, 512)) * 0.05).astype(np.float16)
    W[3, :group] = 0  # an all-zero group -> scale 1, codes 0
    _, Sw32 = oracle.pack_weight(W, group)
    Wq, Sw16 = O.pack_weight_bf16s(W, group)
    assert np.array_equal(Sw16, O.f32_to_bf16_bits(Sw32))
    assert O.bf16_bits_to_f32(Sw16[0, 3]) == 1.0 and not _unpack(Wq)[3, :group].any()


def test_bf16_exact_scales_give_the_o5_codes():
    rng = np.random.default_rng(14)
    W = (rng.integers(-56, 57, size=(8, 256)) / 8.0).astype(np.float16)
    W[:, 0] = 7.0
    W[:, 128] = -7.0
    Wq32, Sw32 = oracle.pack_weight(W, 128)
    Wqb, Swb = O.pack_weight_bf16s(W, 128)
    assert np.array_equal(O.bf16_bits_to_f32(Swb), Sw32) and np.array_equal(Wqb, Wq32)


def test_bf16_round_trip_bound_with_the_clamp():
    # one bf16 rounding of a / 7 (2^-8 relative): |w - s q| <= max(s / 2, a 2^-8)
    rng = np.random.default_rng(15)
    W = (rng.standard_normal((32, 256)) * np.exp(rng.uniform(-6, 3, size=(32, 1)))).astype(np.float16)
    Wq, Swb = O.pack_weight_bf16s(W, 128)
    q = _unpack(Wq).astype(np.float64)
    s = np.repeat(O.bf16_bits_to_f32(Swb).astype(np.float64).T, 128, axis=1)
    w = W.astype(np.float64)
    a = np.repeat(np.abs(w).reshape(32, 2, 128).max(axis=2), 128, axis=1)
    err = np.abs(w - s * q)
    assert np.all(err <= np.maximum(s / 2, a * 2.0 ** -8) * (1 + 2.0 ** -20) + 1e-30)
    assert np.all(np.abs(q) <= 7)


@pytest.mark.gpu
@pytest.mark.parametrize("M,N,K,group", [(16, 256, 512, 128), (300, 640, 1024, 128), (300, 640, 1024, 1024)])
def test_bf16_scales_gpu_parity(M, N, K, group):
    import torch
    from paper_2410_12168_b200 import comet
    p = synth.make_problem(M, N, K, n8=2, seed=17 + M, mask="scattered")
    dev = torch.device("cuda")
    X, W, perm = (torch.from_numpy(p[k]).to(dev) for k in ("X", "W", "perm"))
    bits = comet.BlockBits(p["bits"])
    Wq, Swb = comet.comet_pack_weight_bf16s(W, perm, group)
    oWq, oSwb = O.pack_weight_bf16s(p["W"], group, p["perm"])
    assert np.array_equal(comet.wq_tiled_to_rowmajor(Wq.cpu().numpy(), N, K), oWq)
    assert np.array_equal(Swb.view(torch.int16).cpu().numpy().view(np.uint16), oSwb)
    Xq8, Xq4, Sx = comet.comet_quantize_act(X, bits, perm)
    Y = comet.comet_w4ax_gemm_bf16s(Xq8, Xq4, Sx, bits, Wq, Swb, group)
    ws = comet.new_workspace(comet.comet_w4ax_gemm_workspace_bytes(M, N, K), dev)
    Y32 = comet.comet_w4ax_gemm(Xq8, Xq4, Sx, bits, Wq, Swb.float().contiguous(), group, workspace=ws)
    torch.cuda.synchronize()
    assert np.array_equal(Y.cpu().numpy().view(np.uint16), Y32.cpu().numpy().view(np.uint16))
    o8, o4, os_ = oracle.quantize_act(p["X"], p["bits"], p["perm"])
    ref = oracle.w4ax_gemm(o8, o4, os_, p["bits"], oWq, O.bf16_bits_to_f32(oSwb), group=group)["y"].astype(np.float64)
    y = Y.float().cpu().numpy().astype(np.float64)
    assert np.all(np.abs(y - ref) <= np.maximum(2.0 ** -10 * np.abs(ref), 1e-3))
