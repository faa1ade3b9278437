"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Each test names the pin and
what it fixes.  Sources of truth: hand-worked values (tests/golden/),
library routines (numpy float16 conversion, numpy integer matmul), closed
forms, brute force in exact rational arithmetic, and invariants.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from paper_2410_12168_b200 import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hand_worked.json")))


def _block(head, n=128):
    x = np.zeros(n, np.float32)
    x[: len(head)] = head
    return x


# ---------------------------------------------------------------- fp16 ----
def test_half_to_float_all_patterns_match_numpy():
    """Library-routine pin: every one of the 65536 binary16 patterns."""
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    ref = bits.view(np.float16).astype(np.float32)
    got = np.array([oracle.half_to_float(int(b)) for b in bits], np.float32)
    finite = np.isfinite(ref)
    assert np.array_equal(got[finite].view(np.uint32), ref[finite].view(np.uint32))
    assert np.array_equal(np.isnan(got), np.isnan(ref))
    assert np.array_equal(np.isinf(got), np.isinf(ref))


def test_double_to_half_rne_matches_numpy():
    """Library-routine pin: RNE incl. exact ties, subnormals and overflow."""
    rng = np.random.default_rng(0)
    vals = list(rng.standard_normal(3000) * 10.0 ** rng.uniform(-9, 5, 3000))
    # exact ties between adjacent halves (normal and subnormal), overflow edge
    h = np.arange(0, 0x7BFF, 97, dtype=np.uint16).view(np.float16).astype(np.float64)
    h2 = (np.arange(0, 0x7BFF, 97, dtype=np.uint16) + 1).view(np.float16).astype(np.float64)
    vals += list((h + h2) / 2) + list(-(h + h2) / 2)
    vals += [65504.0, 65519.99, 65520.0, 70000.0, -65520.0, 2.0 ** -25, 3 * 2.0 ** -26, 0.0, -0.0, 1e-30]
    for v in vals:
        with np.errstate(over="ignore"):
            ref = np.array(v, np.float64).astype(np.float16).view(np.uint16)
        assert oracle.double_to_half_bits(v) == int(ref), v


# ------------------------------------------------------ quantization pins ----
def test_P1_int4_block_hand_worked():
    g = GOLD["P1_int4_block"]
    q, s = oracle.quantize_block(_block(g["x_head"]), g["qmax"])
    assert np.float32(s).view(np.uint32) == int(g["s_bits"], 16)
    assert list(q[:8]) == g["q_head"] and not q[8:].any()
    word = int.from_bytes(oracle.pack_int4(q)[:4].tobytes(), "little")
    assert word == int(g["packed_word_le"], 16)
    # the paper's zero-extension: x16 values, 2 word ops
    lo = np.array([(word << 4) & 0xF0F0F0F0], np.uint32).view(np.int8)
    hi = np.array([word & 0xF0F0F0F0], np.uint32).view(np.int8)
    assert list(lo) == g["expand_lo_bytes"] and list(hi) == g["expand_hi_bytes"]


def test_P2_rounding_is_half_away_not_half_even():
    g = GOLD["P1_int4_block"]
    q, _ = oracle.quantize_block(_block(g["x_head"]), 7)
    assert list(q[:8]) != g["q_half_even_head"]
    assert list(np.round(np.float32(2.0) * np.array(g["x_head"], np.float32)).astype(int)) == g["q_half_even_head"]


def test_P3_int8_block_hand_worked_with_fp32_tie():
    g = GOLD["P3_int8_block"]
    x = _block(np.array(g["x_head"], np.float16).astype(np.float32))  # activations are fp16
    q, s = oracle.quantize_block(x, g["qmax"])
    assert np.float32(s).view(np.uint32) == int(g["s_bits"], 16)
    assert list(q[:5]) == g["q_head"] and not q[5:].any()


def test_spec_scale_examples():
    """S:L68 (scale = 14/7 = 2) and S:L77 (x=3.4, scale 1 -> 3)."""
    q, s = oracle.quantize_block(_block([-14.0, 7.0, 3.0]), 7)
    assert s == 2.0 and list(q[:3]) == [-7, 4, 2]  # 3/2 = 1.5 -> 2 (half away)
    q, s = oracle.quantize_block(_block([7.0, 3.4, -3.5, 0.5]), 7)
    assert s == 1.0 and list(q[:4]) == [7, 3, -4, 1]


def test_zero_block_degenerate_scale():
    """A-7 / S:L70: all-zero (and -0) block -> s = 1, q = 0."""
    x = np.zeros(128, np.float32)
    x[3] = -0.0
    q, s = oracle.quantize_block(x, 7)
    assert s == 1.0 and not q.any()


@pytest.mark.parametrize("qmax", [7, 127])
def test_P10_round_trip_bound_and_monotone(qmax):
    rng = np.random.default_rng(qmax)
    for t in range(200):
        x = (rng.standard_normal(128) * 10.0 ** rng.uniform(-3, 3)).astype(np.float16).astype(np.float32)
        q, s = oracle.quantize_block(x, qmax)
        err = np.abs(x.astype(np.float64) - np.float64(s) * q)
        # s/2 in exact arithmetic; x*r with r = fl(qmax/a) deviates from x/s by
        # at most ~qmax * 2^-22 of a step (two fp32 roundings of s and r, one of x*r)
        assert np.all(err <= np.float64(s) * (0.5 + qmax * 2.0 ** -21)), (t, err.max() / s)
        assert np.abs(q).max() <= qmax and np.abs(q).max() == qmax
        o = np.argsort(x, kind="stable")
        assert np.all(np.diff(q[o].astype(int)) >= 0)


# ----------------------------------------------------------- packing pins ----
def test_P5_pack_unpack_exhaustive_and_zero_extension():
    """Every (e_j, e_{j+4}) nibble pair at every byte position; the paper's
    x16 zero-extension recovers 16*e exactly."""
    vals = np.arange(-8, 8)
    pairs = np.array([(a, b) for a in vals for b in vals], np.int8)
    for j in range(4):
        q = np.zeros((len(pairs), 8), np.int8)
        q[:, j] = pairs[:, 0]
        q[:, j + 4] = pairs[:, 1]
        p = oracle.pack_int4(q.reshape(-1)).reshape(-1, 4)
        assert np.array_equal(oracle.unpack_int4(p.reshape(-1), q.size).reshape(q.shape), q)
        w = p.copy().view(np.uint32).reshape(-1)
        lo = ((w << 4) & 0xF0F0F0F0).astype(np.uint32).view(np.int8).reshape(-1, 4)
        hi = (w & 0xF0F0F0F0).astype(np.uint32).view(np.int8).reshape(-1, 4)
        assert np.array_equal(lo.astype(int), 16 * q[:, 0:4].astype(int))
        assert np.array_equal(hi.astype(int), 16 * q[:, 4:8].astype(int))


def test_P5_paper_16bit_swapped_word_exhaustive():
    """The paper's 16-bit form: slots (w3,w1,w2,w0) at bits
    [12-15],[8-11],[4-7],[0-3]; two word ops give (16w0,16w1),(16w2,16w3).
    Our 32-bit byte order restricted to one 16-bit half is this layout with
    (w0,w1,w2,w3) = (e0,e1,e4,e5)."""
    words = np.arange(65536, dtype=np.uint32)
    nib = lambda s: ((words >> s) & 0xF).astype(int)
    sx = lambda v: np.where(v >= 8, v - 16, v)
    w0, w2, w1, w3 = sx(nib(0)), sx(nib(4)), sx(nib(8)), sx(nib(12))
    lo = ((words << 4) & 0xF0F0).astype(np.uint16).view(np.int8).reshape(-1, 2).astype(int)
    hi = (words & 0xF0F0).astype(np.uint16).view(np.int8).reshape(-1, 2).astype(int)
    assert np.array_equal(lo, 16 * np.stack([w0, w1], 1))
    assert np.array_equal(hi, 16 * np.stack([w2, w3], 1))
    # oracle packing of (e0,e1,..,e4,e5,..) puts e0,e4,e1,e5 at nibbles 0,1,2,3
    q = np.zeros((65536, 8), np.int8)
    q[:, 0], q[:, 4], q[:, 1], q[:, 5] = w0, w2, w1, w3
    p = oracle.pack_int4(q.reshape(-1)).reshape(-1, 4)
    assert np.array_equal(p[:, 0].astype(np.uint32) | (p[:, 1].astype(np.uint32) << 8), words)


def test_P6_scale_fold_exact():
    """dequant(16^e q, s/16^e) == dequant(q, s) exactly."""
    rng = np.random.default_rng(6)
    for _ in range(100):
        q = rng.integers(-127, 128, 1000).astype(np.float32)
        s = np.float32(rng.uniform(1e-4, 10))
        for e in (1, 2):
            f = np.float32(16.0 ** e)
            assert np.array_equal((q * f) * (s / f), q * s)


# -------------------------------------------------------------- GEMM pins ----
def _prob(M, N, K, n8, seed, mask="prefix", with_perm=True, k=128):
    return synth.make_problem(M, N, K, n8=n8, seed=seed, mask=mask, with_perm=with_perm, k=k)


def test_P4_single_block_w4a4_hand_worked():
    g1, g4 = GOLD["P1_int4_block"], GOLD["P4_single_block_w4a4"]
    X = _block(g1["x_head"]).astype(np.float16)[None, :]
    W = _block(g4["w_head"]).astype(np.float16)[None, :]
    bits = np.array([4], np.uint8)
    Xq8, Xq4, Sx = oracle.quantize_act(X, bits)
    Wq, Sw = oracle.pack_weight(W, group=128)
    assert Sw[0, 0] == g4["sw"]
    assert list(oracle.unpack_int4(Wq[0], 128)[:8]) == g4["wq_head"]
    r = oracle.w4ax_gemm(Xq8, Xq4, Sx, bits, Wq, Sw, group=128, want_acc=True, want_y64=True)
    assert r["acc"][0, 0, 0] == g4["acc"] and r["y64"][0, 0] == g4["y"] and r["y"][0, 0] == g4["y"]
    assert g4["acc"] * 256 == g4["expanded_acc_x256"]


@pytest.mark.parametrize("group", [128, 512])
def test_P7_all_int8_mask_equals_integer_matmul(group):
    """Library pin: per-block INT32 == numpy int64 matmul; Y64 == dense fp64
    combination; Y == numpy's fp16 rounding of Y64."""
    M, N, K = 16, 64, 512
    p = _prob(M, N, K, n8=4, seed=11)
    bits = p["bits"]
    assert (bits == 8).all()
    Xq8, Xq4, Sx = oracle.quantize_act(p["X"], bits, p["perm"])
    Wq, Sw = oracle.pack_weight(p["W"], group, p["perm"])
    r = oracle.w4ax_gemm(Xq8, Xq4, Sx, bits, Wq, Sw, group=group, want_acc=True, want_y64=True)
    wq = np.stack([oracle.unpack_int4(Wq[n], K) for n in range(N)]).astype(np.int64)
    x = Xq8.astype(np.int64)
    y = np.zeros((M, N))
    for b in range(K // 128):
        acc = x[:, b * 128:(b + 1) * 128] @ wq[:, b * 128:(b + 1) * 128].T
        assert np.array_equal(r["acc"][b], acc)
        y += Sx[b, :M, None].astype(np.float64) * Sw[(b * 128) // group][None, :].astype(np.float64) * acc
    np.testing.assert_allclose(r["y64"], y, rtol=1e-13, atol=1e-13)
    assert np.array_equal(r["y"].view(np.uint16), r["y64"].astype(np.float16).view(np.uint16))


def test_end_to_end_equals_dense_fp64_of_dequantized_operands():
    """Y64 == f64 matmul of dequantized (permuted) operands."""
    M, N, K = 32, 128, 1024
    p = _prob(M, N, K, n8=2, seed=5, mask="scattered")
    Xq8, Xq4, Sx = oracle.quantize_act(p["X"], p["bits"], p["perm"])
    Wq, Sw = oracle.pack_weight(p["W"], 128, p["perm"])
    r = oracle.w4ax_gemm(Xq8, Xq4, Sx, p["bits"], Wq, Sw, group=128, want_y64=True)
    # dequantize both operands onto the permuted axis
    xd = np.zeros((M, K))
    r8 = r4 = 0
    for b, bb in enumerate(p["bits"]):
        if bb == 8:
            q = Xq8[:, r8 * 128:(r8 + 1) * 128].astype(np.float64); r8 += 1
        else:
            q = np.stack([oracle.unpack_int4(Xq4[m, r4 * 64:(r4 + 1) * 64], 128) for m in range(M)]).astype(np.float64); r4 += 1
        xd[:, b * 128:(b + 1) * 128] = q * Sx[b, :M, None]
    wd = np.stack([oracle.unpack_int4(Wq[n], K) for n in range(N)]).astype(np.float64)
    wd *= np.repeat(Sw.T.astype(np.float64), 128, axis=1)
    ref = xd @ wd.T
    assert np.linalg.norm(r["y64"] - ref) <= 1e-12 * np.linalg.norm(ref)
    # and the quantized GEMM approximates the unquantized one (sanity, not exactness)
    exact = p["X"].astype(np.float64) @ p["W"].astype(np.float64).T
    assert np.linalg.norm(r["y64"] - exact) <= 0.2 * np.linalg.norm(exact)


def test_P8_permutation_equivalence():
    """Fused gather == pre-permuted input."""
    M, N, K = 8, 128, 512
    p = _prob(M, N, K, n8=1, seed=3)
    perm = p["perm"]
    a = oracle.quantize_act(p["X"], p["bits"], perm)
    b = oracle.quantize_act(np.ascontiguousarray(p["X"][:, perm]), p["bits"], None)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)
    wa = oracle.pack_weight(p["W"], 128, perm)
    wb = oracle.pack_weight(np.ascontiguousarray(p["W"][:, perm]), 128, None)
    for u, v in zip(wa, wb):
        assert np.array_equal(u, v)
    # permuting both operands' reduction axis preserves the exact product
    xi = np.random.default_rng(1).integers(-7, 8, (8, 16))
    wi = np.random.default_rng(2).integers(-7, 8, (8, 16))
    pp = np.random.default_rng(3).permutation(16)
    assert np.array_equal(xi @ wi.T, xi[:, pp] @ wi[:, pp].T)


def _brute_force(X, W, bits, k, group):
    """Triple loop in exact rational arithmetic on dequantized values, with
    quantization re-derived per element from the block scale."""
    M, K = X.shape
    N = W.shape[0]
    Xf = X.astype(np.float32)
    Wf = W.astype(np.float32)

    def quant(vals, qmax):
        a = np.float32(max(abs(float(v)) for v in vals))
        if a == 0:
            return [0] * len(vals), np.float32(1.0)
        s = np.float32(a / np.float32(qmax))
        r = np.float32(np.float32(qmax) / a)
        out = []
        for v in vals:
            t = float(np.float32(v * r))
            qi = int(Fraction(abs(t)) + Fraction(1, 2))  # floor(|t| + 1/2)
            out.append(max(-qmax, min(qmax, qi if t >= 0 else -qi)))
        return out, s

    xq = [[None] * (K // k) for _ in range(M)]
    wq = [[None] * (K // group) for _ in range(N)]
    for m in range(M):
        for b in range(K // k):
            xq[m][b] = quant(Xf[m, b * k:(b + 1) * k], 7 if bits[b] == 4 else 127)
    for n in range(N):
        for j in range(K // group):
            wq[n][j] = quant(Wf[n, j * group:(j + 1) * group], 7)
    Y = np.zeros((M, N))
    for m in range(M):
        for n in range(N):
            tot = Fraction(0)
            for i in range(K):
                qx, sx = xq[m][i // k]
                qw, sw = wq[n][i // group]
                tot += Fraction(float(sx)) * qx[i % k] * Fraction(float(sw)) * qw[i % group]
            Y[m, n] = float(tot)
    return Y


@pytest.mark.parametrize("bits", [[4], [8]])
def test_P9_brute_force_8x8x64(bits):
    """BJ north_star: brute force on 8x8x64 inputs (oracle block size k=64)."""
    rng = np.random.default_rng(9)
    X = (rng.standard_normal((8, 64)) * 3).astype(np.float16)
    X[2, 5] = 40.0  # an outlier channel
    W = (rng.standard_normal((8, 64)) / 8).astype(np.float16)
    b = np.array(bits, np.uint8)
    Xq8, Xq4, Sx = oracle.quantize_act(X, b, None, k=64)
    Wq, Sw = oracle.pack_weight(W, group=64)
    r = oracle.w4ax_gemm(Xq8, Xq4, Sx, b, Wq, Sw, group=64, k=64, want_y64=True)
    ref = _brute_force(X, W, b, 64, 64)
    np.testing.assert_allclose(r["y64"], ref, rtol=1e-12, atol=1e-12)


def test_P9_zero_padding_to_abi_shape_is_identical():
    """A-18: an 8x8x64 problem zero-padded to M=8, N=128, K=128 (k=128)
    gives the same Y in the 8x8 corner as the k=64 oracle."""
    rng = np.random.default_rng(10)
    X = (rng.standard_normal((8, 64)) * 2).astype(np.float16)
    W = (rng.standard_normal((8, 64)) / 8).astype(np.float16)
    b64 = np.array([4], np.uint8)
    r64 = oracle.w4ax_gemm(*oracle.quantize_act(X, b64, None, k=64), b64, *oracle.pack_weight(W, 64), group=64, k=64, want_y64=True)
    Xp = np.zeros((8, 128), np.float16); Xp[:, :64] = X
    Wp = np.zeros((128, 128), np.float16); Wp[:8, :64] = W
    b128 = np.array([4], np.uint8)
    r128 = oracle.w4ax_gemm(*oracle.quantize_act(Xp, b128), b128, *oracle.pack_weight(Wp, 128), group=128, want_y64=True)
    assert np.array_equal(r128["y64"][:, :8], r64["y64"])
    assert not r128["y64"][:, 8:].any()


def test_P11_power_of_two_scales_exact():
    """Integer data with block absmax = qmax * 2^e: quantization is exact, so
    Y64 equals the exact product X . W^T (numpy fp64 on small integers)."""
    rng = np.random.default_rng(12)
    M, N, K = 8, 128, 256
    bits = np.array([8, 4], np.uint8)
    X = rng.integers(-7, 8, (M, K)).astype(np.float64)
    X[:, :128] = rng.integers(-127, 128, (M, 128))
    X[:, 0], X[:, 128] = 127, 7
    X[:, :128] *= 0.25
    W = rng.integers(-7, 8, (N, K)).astype(np.float64) * 0.5
    W[:, 0] = 7 * 0.5
    W[:, 128] = -7 * 0.5
    Xq8, Xq4, Sx = oracle.quantize_act(X.astype(np.float16), bits)
    Wq, Sw = oracle.pack_weight(W.astype(np.float16), 128)
    r = oracle.w4ax_gemm(Xq8, Xq4, Sx, bits, Wq, Sw, want_y64=True)
    assert np.array_equal(r["y64"], X @ W.T)


def test_P12_row_independence_and_row_sampling():
    M, N, K = 24, 128, 512
    p = _prob(M, N, K, n8=1, seed=13)
    Xq8, Xq4, Sx = oracle.quantize_act(p["X"], p["bits"], p["perm"])
    Wq, Sw = oracle.pack_weight(p["W"], 128, p["perm"])
    full = oracle.w4ax_gemm(Xq8, Xq4, Sx, p["bits"], Wq, Sw, want_acc=True)
    for m in (0, 7, 23):
        one = oracle.quantize_act(p["X"][m:m + 1], p["bits"], p["perm"])
        assert np.array_equal(one[0][0], Xq8[m]) and np.array_equal(one[1][0], Xq4[m])
        assert np.array_equal(one[2][:, 0], Sx[:, m])
    rows = np.array([23, 0, 5], np.int32)
    sub = oracle.w4ax_gemm(Xq8, Xq4, Sx, p["bits"], Wq, Sw, rows=rows, want_acc=True)
    assert np.array_equal(sub["y"], full["y"][rows])
    assert np.array_equal(sub["acc"], full["acc"][:, rows])


def test_sx_padding_and_plane_layout():
    """A-19: Sx rows beyond M are 1.0; INT8 blocks fill plane8 in block order."""
    M, K = 5, 512
    p = _prob(M, 128, K, n8=2, seed=2, mask=[4, 8, 4, 8], with_perm=False)
    Xq8, Xq4, Sx = oracle.quantize_act(p["X"], p["bits"])
    assert Xq8.shape == (5, 256) and Xq4.shape == (5, 128) and Sx.shape == (4, 8)
    assert (Sx[:, 5:] == 1.0).all()
    q, s = oracle.quantize_block(p["X"][2, 384:512].astype(np.float32), 127)
    assert np.array_equal(Xq8[2, 128:256], q) and Sx[3, 2] == s


def test_weight_error_matches_uniform_rounding_model():
    """Closed form: for dense Gaussian weights the INT4 round-trip error is
    uniform on [-s/2, s/2], so E[e^2] = E[s^2]/12 (per group and per
    channel).  (SPEC's ">= 20 dB" example does not hold for qmax = 7 on
    Gaussian data: the model gives ~18.7 dB, which is what we assert.)"""
    W = np.random.default_rng(4).standard_normal((256, 256)).astype(np.float16)
    for group in (128, 256):
        Wq, Sw = oracle.pack_weight(W, group)
        wd = np.stack([oracle.unpack_int4(Wq[n], 256) for n in range(256)]).astype(np.float64)
        s_el = np.repeat(Sw.T.astype(np.float64), group, axis=1)
        e = W.astype(np.float64) - wd * s_el
        ratio = (e ** 2).mean() / (s_el ** 2 / 12).mean()
        assert 0.9 < ratio < 1.1, ratio
        sqnr = 10 * np.log10((W.astype(np.float64) ** 2).sum() / (e ** 2).sum())
        assert 17.5 < sqnr < 20.0


def test_fmpq_beats_uniform_int4_on_outlier_tensor():
    """S:L206 / S:L573: with outliers clustered into an INT8 block, FMPQ's
    quantization SQNR exceeds all-INT4 on the same (permuted) tensor."""
    p = _prob(16, 128, 512, n8=1, seed=21)
    def sqnr(bits):
        Xq8, Xq4, Sx = oracle.quantize_act(p["X"], bits, p["perm"])
        xp = p["X"][:, p["perm"]].astype(np.float64)
        xd = np.zeros_like(xp); r8 = r4 = 0
        for b, bb in enumerate(bits):
            if bb == 8:
                q = Xq8[:, r8 * 128:(r8 + 1) * 128].astype(np.float64); r8 += 1
            else:
                q = np.stack([oracle.unpack_int4(Xq4[m, r4 * 64:(r4 + 1) * 64], 128) for m in range(16)]); r4 += 1
            xd[:, b * 128:(b + 1) * 128] = q * Sx[b, :16, None]
        return 10 * np.log10((xp ** 2).sum() / ((xp - xd) ** 2).sum())
    assert sqnr(p["bits"]) > sqnr(np.full(4, 4, np.uint8)) + 3.0


def test_errors_on_bad_inputs():
    X = np.zeros((2, 128), np.float16)
    with pytest.raises(oracle.OracleError):
        oracle.quantize_act(X, np.array([5], np.uint8))
    X[0, 0] = np.inf
    with pytest.raises(oracle.OracleError):
        oracle.quantize_act(X, np.array([4], np.uint8))
    with pytest.raises(oracle.OracleError):
        oracle.quantize_act(np.zeros((2, 128), np.float16), np.array([4], np.uint8), perm=np.zeros(128, np.int32))
