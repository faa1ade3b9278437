"""f4: bf16 activations into the W4Ax path.

CPU: the oracle (oracle/fmpq_aux.quantize_act_bf16) pinned to the fp16
oracle on values both formats represent exactly, to exact bf16 -> fp32
decoding, and to bf16-only magnitudes.  GPU: comet_quantize_act_bf16 planes
and Sx bit-exact against it (both the small-M and the row-staged kernels),
and the GEMM on those planes within the Y tolerance.
"""
import numpy as np
import pytest

import oracle
from oracle import fmpq_aux as O


def _bf16_bits(x32: np.ndarray) -> np.ndarray:
    """round-to-nearest-even fp32 -> bf16 encoding (test input generator)."""
    u = np.asarray(x32, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def test_bf16_decoding_exact():
    vals = np.array([0.0, -0.0, 1.0, -2.5, 3.0e38, 1.0e-38, 65504.0, 1.0e6], np.float32)
    b = _bf16_bits(vals)
    back = O.bf16_bits_to_f32(b)
    # every bf16 encoding is an fp32 value: decode(encode(v)) is v rounded to 8 mantissa bits
    assert back[2] == 1.0 and back[3] == -2.5 and back[6] == 65536.0 and np.signbit(back[1])
    assert np.array_equal(_bf16_bits(back), b)


def test_equals_fp16_oracle_on_shared_values():
    # values on a grid both fp16 and bf16 represent exactly (8 significant bits, small exponents)
    rng = np.random.default_rng(0)
    M, K = 5, 512
    bits = np.array([8, 4, 4, 4], np.uint8)
    X = (rng.integers(-255, 256, (M, K)) * 2.0 ** rng.integers(-8, 2, (M, K))).astype(np.float32)
    assert np.array_equal(X.astype(np.float16).astype(np.float32), X)
    assert np.array_equal(O.bf16_bits_to_f32(_bf16_bits(X)), X)
    perm = rng.permutation(K).astype(np.int32)
    got = O.quantize_act_bf16(_bf16_bits(X), bits, perm)
    ref = oracle.quantize_act(X.astype(np.float16), bits, perm)
    for g, r in zip(got, ref):
        assert np.array_equal(g, r)


def test_bf16_only_magnitudes():
    # 1e6 is beyond fp16: the block scale follows the bf16 value
    M, K = 1, 128
    X = np.zeros((M, K), np.float32)
    X[0, 0] = 1.0e6
    X[0, 1] = -5.0e5
    b = _bf16_bits(X)
    x0 = O.bf16_bits_to_f32(b)[0, 0]
    Xq8, Xq4, Sx = O.quantize_act_bf16(b, [8])
    assert Sx[0, 0] == np.float32(x0 / np.float32(127.0))
    assert Xq8[0, 0] == 127 and Xq8[0, 1] == -63 and np.all(Xq8[0, 2:] == 0)  # -499712 / 999424 * 127 = -63.5 -> -63 (the fp32 product rounds below the tie)


@pytest.mark.gpu
@pytest.mark.parametrize("M,K,use_perm", [(1, 128, False), (37, 1024, True), (300, 2048, True)])
def test_bf16_quantize_bit_exact(M, K, use_perm):
    import torch
    from paper_2410_12168_b200 import comet

    rng = np.random.default_rng(M + K)
    nb = K // 128
    bits = np.full(nb, 4, np.uint8)
    bits[rng.choice(nb, max(1, nb // 8), replace=False)] = 8
    X32 = rng.standard_normal((M, K)).astype(np.float32)
    X32[:, rng.integers(0, K, 3)] *= 3.0e5  # beyond fp16 range
    b16 = _bf16_bits(X32)
    perm = rng.permutation(K).astype(np.int32) if use_perm else None
    dev = torch.device("cuda")
    Xd = torch.from_numpy(b16.view(np.int16)).to(dev).view(torch.bfloat16)
    perm_d = None if perm is None else torch.from_numpy(perm).to(dev)
    Xq8, Xq4, Sx = comet.comet_quantize_act_bf16(Xd, bits, perm_d)
    r8, r4, rs = O.quantize_act_bf16(b16, bits, perm)
    assert np.array_equal(Xq8.cpu().numpy(), r8)
    assert np.array_equal(Xq4.cpu().numpy(), r4)
    assert np.array_equal(Sx.cpu().numpy(), rs)


@pytest.mark.gpu
def test_bf16_planes_through_the_gemm():
    import torch
    from paper_2410_12168_b200 import comet

    rng = np.random.default_rng(9)
    M, N, K = 300, 256, 1024
    bits = np.array([8, 4, 4, 4, 4, 4, 4, 4], np.uint8)
    b16 = _bf16_bits(rng.standard_normal((M, K)).astype(np.float32))
    W = (rng.standard_normal((N, K)) * 0.05).astype(np.float16)
    dev = torch.device("cuda")
    Xq8, Xq4, Sx = comet.comet_quantize_act_bf16(torch.from_numpy(b16.view(np.int16)).to(dev).view(torch.bfloat16), bits)
    Wq, Sw = comet.comet_pack_weight(torch.from_numpy(W).to(dev), None, 128)
    ws = comet.new_workspace(comet.comet_w4ax_gemm_workspace_bytes(M, N, K), dev)
    Y = comet.comet_w4ax_gemm(Xq8, Xq4, Sx, bits, Wq, Sw, 128, workspace=ws).float().cpu().numpy()
    r8, r4, rs = O.quantize_act_bf16(b16, bits)
    Wq_o, Sw_o = oracle.pack_weight(W, 128)
    ref = oracle.w4ax_gemm(r8, r4, rs, bits, Wq_o, Sw_o, 128)["y"].astype(np.float32)
    assert np.all(np.abs(Y - ref) <= np.maximum(2.0 ** -10 * np.abs(ref), 1e-3))
