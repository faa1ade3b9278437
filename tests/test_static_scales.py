"""f4: static per-block activation scales.

CPU: the oracle (oracle/fmpq_aux.static_block_scales, quantize_act_static)
pinned to SPEC's worked examples (compute_scale and quantize),
lattice round trips, the round-trip bound, clamping and an end-to-end GEMM
bound.  GPU: comet_static_act_scales / comet_quantize_act_static bit-exact
against the oracle, and the W4Ax GEMM on statically quantized planes.
"""
import numpy as np
import pytest

import oracle
from oracle import fmpq_aux as O


def test_spec_compute_scale_example():
    # S:L66 "min=-14, max=7, b=4, symmetric -> scale = 2.0 (=14/7)"
    maxabs = np.ones(128, np.float32)
    maxabs[5] = 14.0
    assert O.static_block_scales(maxabs, [4])[0] == np.float32(2.0)
    # 8-bit block: qmax 127
    assert O.static_block_scales(maxabs, [8])[0] == np.float32(np.float32(14.0) / np.float32(127.0))
    # degenerate (all-zero calibration) -> scale 1
    assert O.static_block_scales(np.zeros(256, np.float32), [4, 8]).tolist() == [1.0, 1.0]


def test_scales_pool_over_the_permuted_block():
    K = 256
    maxabs = np.ones(K, np.float32)
    maxabs[200] = 70.0  # original channel 200 sits in block 0 after the permutation
    perm = np.r_[200, np.delete(np.arange(K), 200)].astype(np.int32)
    s = O.static_block_scales(maxabs, [8, 4], perm)
    assert s[0] == np.float32(np.float32(70.0) / np.float32(127.0))
    assert s[1] == np.float32(np.float32(1.0) / np.float32(7.0))
    s_id = O.static_block_scales(maxabs, [8, 4])  # identity: the outlier is in block 1
    assert s_id[1] == np.float32(10.0)


def test_spec_quantize_examples():
    # x=3.4, scale=1 -> 3; x=100, scale=1 -> 7 (clamped); symmetric 4-bit
    assert O._q_static(np.float32(3.4), np.float32(1.0), 7) == 3
    assert O._q_static(np.float32(100.0), np.float32(1.0), 7) == 7
    assert O._q_static(np.float32(-100.0), np.float32(1.0), 7) == -7
    assert O._q_static(np.float32(2.5), np.float32(1.0), 7) == 3  # half away from zero
    assert O._q_static(np.float32(-2.5), np.float32(1.0), 7) == -3
    assert O._q_static(np.float32(300.0), np.float32(1.0), 127) == 127


def test_lattice_round_trip_exact():
    # x = s * q on the lattice (s a power of two: every product exact in fp16)
    rng = np.random.default_rng(0)
    M, K = 3, 256
    bits = [4, 8]
    scales = np.array([0.25, 0.5], np.float32)
    q4 = rng.integers(-7, 8, (M, 128))
    q8 = rng.integers(-127, 128, (M, 128))
    X = np.concatenate([q4 * 0.25, q8 * 0.5], axis=1).astype(np.float16)
    Xq8, Xq4, Sx = O.quantize_act_static(X, bits, scales)
    assert np.array_equal(Xq8.astype(np.int64), q8)
    assert np.array_equal(oracle.unpack_int4(Xq4.reshape(-1), M * 128).reshape(M, 128).astype(np.int64), q4)
    assert np.all(Sx[0, :M] == 0.25) and np.all(Sx[1, :M] == 0.5) and np.all(Sx[:, M:] == 1.0)


def test_round_trip_bound_and_clamp():
    rng = np.random.default_rng(1)
    M, K = 5, 384
    bits = [4, 8, 4]
    X = rng.standard_normal((M, K)).astype(np.float16)
    cal = np.abs(X[:2].astype(np.float32)).max(axis=0)  # calibration on 2 of the 5 rows
    scales = O.static_block_scales(cal, bits)
    Xq8, Xq4, Sx = O.quantize_act_static(X, bits, scales)
    q4 = oracle.unpack_int4(Xq4.reshape(-1), M * 256).reshape(M, 256).astype(np.float64)
    q = np.concatenate([q4[:, :128], Xq8.astype(np.float64), q4[:, 128:]], axis=1)
    s = np.repeat(scales.astype(np.float64), 128)
    qmax = np.repeat([7.0, 127.0, 7.0], 128)
    x = X.astype(np.float64)
    inside = np.abs(x) <= qmax * s
    err = np.abs(q * s - x)
    # s/2, plus the fp32 rounding of the quotient x/s (a tie can round away)
    cols = np.nonzero(inside)[1]
    assert np.all(err[inside] <= s[cols] / 2 + np.abs(x[inside]) * 2.0 ** -23)
    # outside the calibrated range: clamped to +-qmax with the sign of x
    out = ~inside
    assert np.all(np.abs(q[out]) == qmax[np.nonzero(out)[1]])
    assert np.all(np.sign(q[out]) == np.sign(x[out]))
    # rows used for calibration never clamp beyond the bound
    assert np.all(inside[:2])


def test_static_equals_dynamic_when_calibrated_on_the_row():
    # one token row whose own absmax is the calibration: the static scale is
    # the dynamic one (a / qmax), and the integers agree with the dynamic
    # oracle except where x*(qmax/a) and x/(a/qmax) round to different sides
    # of a tie (never more than 1 apart)
    rng = np.random.default_rng(2)
    K = 1024
    bits = np.array([8, 4, 4, 4, 4, 4, 4, 4], np.uint8)
    X = rng.standard_normal((1, K)).astype(np.float16)
    scales = O.static_block_scales(np.abs(X[0].astype(np.float32)), bits)
    s8, s4, ss = O.quantize_act_static(X, bits, scales)
    d8, d4, ds = oracle.quantize_act(X, bits)
    assert np.array_equal(ss, ds)
    qs = np.r_[s8[0].astype(np.int64), oracle.unpack_int4(s4[0], 896).astype(np.int64)]
    qd = np.r_[d8[0].astype(np.int64), oracle.unpack_int4(d4[0], 896).astype(np.int64)]
    assert np.abs(qs - qd).max() <= 1
    assert (qs == qd).mean() >= 0.99


def test_static_gemm_error_matches_dynamic():
    rng = np.random.default_rng(3)
    M, N, K = 4, 128, 256
    bits = [8, 4]
    X = rng.standard_normal((M, K)).astype(np.float16)
    W = (rng.standard_normal((N, K)) * 0.05).astype(np.float16)
    scales = O.static_block_scales(np.abs(X.astype(np.float32)).max(axis=0), bits)
    Wq, Sw = oracle.pack_weight(W, 128)
    ref = X.astype(np.float64) @ W.astype(np.float64).T
    Ys = oracle.w4ax_gemm(*O.quantize_act_static(X, bits, scales), bits, Wq, Sw, 128)["y"].astype(np.float64)
    Yd = oracle.w4ax_gemm(*oracle.quantize_act(X, bits), bits, Wq, Sw, 128)["y"].astype(np.float64)
    # pooled (per-block, all rows) scales are >= each row's own: the error
    # stays within a small factor of the dynamic path's
    es, ed = np.sqrt(np.mean((Ys - ref) ** 2)), np.sqrt(np.mean((Yd - ref) ** 2))
    assert es <= 2.0 * ed


# ---------------------------------------------------------------- GPU ----
@pytest.mark.gpu
@pytest.mark.parametrize("M,K,use_perm", [(1, 128, False), (37, 1024, True), (300, 2048, True), (4096, 4096, False)])
def test_static_quantize_bit_exact(M, K, use_perm):
    import torch
    from paper_2410_12168_b200 import comet

    rng = np.random.default_rng(M + K)
    nb = K // 128
    bits = np.full(nb, 4, np.uint8)
    bits[rng.choice(nb, max(1, nb // 8), replace=False)] = 8
    X = rng.standard_normal((M, K)).astype(np.float16)
    X[:, rng.integers(0, K, 3)] *= 40.0  # outlier channels
    perm = rng.permutation(K).astype(np.int32) if use_perm else None
    ncal = max(1, M // 2)
    cal = np.abs(X[:ncal].astype(np.float32)).max(axis=0)
    dev = torch.device("cuda")
    maxabs_d = torch.from_numpy(cal).to(dev)
    perm_d = None if perm is None else torch.from_numpy(perm).to(dev)
    scales = comet.comet_static_act_scales(maxabs_d, bits, perm_d)
    ref_s = O.static_block_scales(cal, bits, perm)
    assert np.array_equal(scales.cpu().numpy().view(np.uint32), ref_s.view(np.uint32))
    Xq8, Xq4, Sx = comet.comet_quantize_act_static(torch.from_numpy(X).to(dev), bits, scales, perm_d)
    if M * K <= 300 * 2048:
        r8, r4, rs = O.quantize_act_static(X, bits, ref_s, perm)
        rows = np.arange(M)
    else:  # full size: sampled rows through the oracle
        rows = np.sort(rng.choice(M, 16, replace=False))
        r8, r4, rs = O.quantize_act_static(X[rows], bits, ref_s, None if perm is None else perm)
    g8 = Xq8.cpu().numpy()[rows] if Xq8 is not None else np.zeros((len(rows), 0), np.int8)
    g4 = Xq4.cpu().numpy()[rows] if Xq4 is not None else np.zeros((len(rows), 0), np.uint8)
    assert np.array_equal(g8, r8)
    assert np.array_equal(g4, r4)
    assert np.array_equal(Sx.cpu().numpy()[:, rows], rs[:, :len(rows)])


@pytest.mark.gpu
def test_static_planes_through_the_gemm():
    import torch
    from paper_2410_12168_b200 import comet

    rng = np.random.default_rng(7)
    M, N, K = 300, 256, 1024
    bits = np.array([8, 4, 4, 4, 4, 4, 4, 4], np.uint8)
    X = rng.standard_normal((M, K)).astype(np.float16)
    W = (rng.standard_normal((N, K)) * 0.05).astype(np.float16)
    dev = torch.device("cuda")
    scales_np = O.static_block_scales(np.abs(X.astype(np.float32)).max(axis=0), bits)
    scales = torch.from_numpy(scales_np).to(dev)
    Xq8, Xq4, Sx = comet.comet_quantize_act_static(torch.from_numpy(X).to(dev), bits, scales)
    Wq, Sw = comet.comet_pack_weight(torch.from_numpy(W).to(dev), None, 128)
    ws = comet.new_workspace(comet.comet_w4ax_gemm_workspace_bytes(M, N, K), dev)
    Y = comet.comet_w4ax_gemm(Xq8, Xq4, Sx, bits, Wq, Sw, 128, workspace=ws).float().cpu().numpy()
    r8, r4, rs = O.quantize_act_static(X, bits, scales_np)
    Wq_o, Sw_o = oracle.pack_weight(W, 128)
    ref = oracle.w4ax_gemm(r8, r4, rs, bits, Wq_o, Sw_o, 128)["y"].astype(np.float32)
    tol = np.maximum(2.0 ** -10 * np.abs(ref), 1e-3)
    assert np.all(np.abs(Y - ref) <= tol)
