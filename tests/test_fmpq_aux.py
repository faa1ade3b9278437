"""f2 (calibration -> permutation + block mask) and f3 (KV4 cache) -- SURVEY 8(f).

-m "not gpu": the oracle (oracle/fmpq_aux.py) against the SPEC's worked
examples and closed-form properties, and the library's host-side map builder
(comet_fmpq_map in libcomet.so, no GPU needed) against the oracle.
-m gpu: the calibration and KV4 kernels against the oracle, bit-exact.
"""
import numpy as np
import pytest

from oracle import fmpq_aux as O


# --------------------------------------------------------- oracle pins ----
def test_detect_outliers_spec_examples():
    # scores [1,1,1,100], theta 8 -> median 1 (lower middle), outliers {3}
    assert list(np.nonzero(O.detect_outliers(np.array([1, 1, 1, 100], np.float32)))[0]) == [3]
    # all equal -> none
    assert not O.detect_outliers(np.full(64, 3.5, np.float32)).any()
    # lower-middle median for even C: [1, 2, 30, 40] -> median 2, threshold 16 -> {2, 3}
    assert list(np.nonzero(O.detect_outliers(np.array([1, 2, 30, 40], np.float32)))[0]) == [2, 3]


def test_planted_outliers_are_found_exactly():
    # 512 Gaussian channels + 5 planted x50 channels, theta 8 -> exactly the 5
    rng = np.random.default_rng(0)
    X = rng.standard_normal((256, 512)).astype(np.float16)
    planted = [7, 100, 255, 256, 500]
    X[:, planted] = (X[:, planted].astype(np.float32) * 50).astype(np.float16)
    flags = O.detect_outliers(O.calib_absmax(X))
    assert sorted(np.nonzero(flags)[0].tolist()) == planted


def test_build_permutation_spec_examples():
    # outliers {3, 200, 450} scores 100, 90, 80 -> perm starts [3, 200, 450], 8-bit set {0}
    score = np.ones(512, np.float32)
    score[[3, 200, 450]] = [100, 90, 80]
    perm, bits, n = O.fmpq_map(score)
    assert perm[:3].tolist() == [3, 200, 450] and n == 3
    rest = [c for c in range(512) if c not in (3, 200, 450)]
    assert perm[3:].tolist() == rest  # stable
    assert bits.tolist() == [8, 4, 4, 4]
    # no outliers -> identity
    perm, bits, n = O.fmpq_map(np.ones(256, np.float32))
    assert perm.tolist() == list(range(256)) and bits.tolist() == [4, 4] and n == 0
    # 140 outliers, k = 128 -> 8-bit blocks {0, 1}
    score = np.ones(512, np.float32)
    score[np.arange(140) * 3] = 50.0
    _, bits, n = O.fmpq_map(score)
    assert n == 140 and bits.tolist() == [8, 8, 4, 4]
    # ties in score: ascending channel index
    score = np.ones(256, np.float32)
    score[[9, 4, 200]] = 20.0
    perm, _, _ = O.fmpq_map(score)
    assert perm[:3].tolist() == [4, 9, 200]


def test_permutation_is_a_bijection_and_minimises_int8_blocks():
    rng = np.random.default_rng(1)
    score = rng.uniform(1, 2, 1024).astype(np.float32)
    idx = rng.choice(1024, 37, replace=False)
    score[idx] *= 40
    perm, bits, n = O.fmpq_map(score)
    assert sorted(perm.tolist()) == list(range(1024))
    assert n == 37 and int((bits == 8).sum()) == 1  # ceil(37 / 128), the pigeonhole minimum


def test_kv_lattice_round_trips():
    # channel values 0..15 -> scale 1, zp 0, exact; -8..7 -> scale 1, zp 8, exact
    T = 16
    KV = np.stack([np.arange(16), np.arange(-8, 8), np.full(16, 2.5), np.zeros(16)], axis=1).astype(np.float16)
    q, s, z = O.quantize_kv(KV, group=T)
    assert s[0, 0] == 1 and z[0, 0] == 0 and s[0, 1] == 1 and z[0, 1] == 8
    assert q[:, 0].tolist() == list(range(16)) and q[:, 1].tolist() == list(range(16))
    y = O.dequantize_kv(q, s, z, T)
    assert np.array_equal(y[:, :2], KV[:, :2])
    # constant channels (degenerate params, exact round trip), incl. negative and zero
    assert s[0, 2] == np.float32(2.5) and z[0, 2] == 0 and np.array_equal(y[:, 2], KV[:, 2])
    assert s[0, 3] == 1 and z[0, 3] == 0 and np.array_equal(y[:, 3], KV[:, 3])
    neg = np.full((8, 2), -3.25, np.float16)
    q, s, z = O.quantize_kv(neg, group=8)
    assert z[0, 0] == 1 and np.array_equal(O.dequantize_kv(q, s, z, 8), neg)


def test_kv_round_trip_bound_and_vectorised_form():
    # S:L191 / S:L91: |x - dq(q(x))| <= scale/2 per element (+ fp32/fp16 rounding of the product)
    rng = np.random.default_rng(2)
    KV = (rng.uniform(-3, 5, (40, 24))).astype(np.float16)
    q, s, z = O.quantize_kv(KV, group=16)
    qv, sv, zv = O.quantize_kv_vec(KV, group=16)
    assert np.array_equal(q, qv) and np.array_equal(s.view(np.uint32), sv.view(np.uint32)) and np.array_equal(z, zv)
    assert q.max() <= 15
    y = O.dequantize_kv(q, s, z, 16).astype(np.float64)
    g = np.arange(40) // 16
    x = KV.astype(np.float64)
    sg, zg = s[g].astype(np.float64), z[g].astype(np.float64)
    slack = np.abs(x) * 2.0 ** -10 + 1e-7  # fp16 rounding of the dequantised value
    # S:L91 "for in-range x": inside the representable grid [-zp*s, (15-zp)*s] the
    # error is <= s/2; the rounded zero point can leave the extreme values of the
    # channel up to s/2 outside the grid, where the clamp bounds the error by s
    inside = (x >= -zg * sg) & (x <= (15 - zg) * sg)
    err = np.abs(y - x)
    assert np.all(err[inside] <= (sg / 2 * (1 + 1e-6) + slack)[inside])
    assert np.all(err <= sg * (1 + 1e-6) + slack)
    # monotone in x within a channel
    col = np.sort(KV[:16, 0].astype(np.float32))
    qq, _, _ = O.quantize_kv(col.astype(np.float16)[:, None].repeat(2, 1), group=16)
    assert np.all(np.diff(qq[:, 0].astype(int)) >= 0)


def test_pack_kv_nibble_order():
    q = np.array([[1, 2, 15, 0]], np.uint8)
    assert O.pack_kv(q).tolist() == [[0x21, 0x0F]]


# ------------------------------------ library host map builder (no GPU) ----
def _lib_map(score, theta=8.0):
    from paper_2410_12168_b200 import comet
    return comet.comet_fmpq_map(score, theta)


# ---------------------------------- f3: attention over the KV4 cache ----
def _kv4_cache(T, C, G, rng, scale=1.0):
    x = (rng.standard_normal((T, C)) * scale).astype(np.float16)
    q, s, z = O.quantize_kv_vec(x, G)
    return O.pack_kv(q), s, z


def test_attention_kv4_single_token_returns_its_value():
    # T = 1: the softmax of one score is 1, so o = V^[0] for any query
    rng = np.random.default_rng(0)
    K, V = _kv4_cache(1, 256, 128, rng), _kv4_cache(1, 256, 128, rng)
    q = rng.standard_normal((2, 128)).astype(np.float16)
    o = O.attention_kv4(q, K, V, 128, 0.088)
    Vh = O.dequantize_kv(O.unpack_kv(V[0]), V[1], V[2], 128).astype(np.float64)
    assert np.array_equal(o, Vh[0].reshape(2, 128))


def test_attention_kv4_zero_query_is_the_mean_value():
    # q = 0: every score is 0, the softmax is uniform, o = mean_t V^[t]
    rng = np.random.default_rng(1)
    T = 37
    K, V = _kv4_cache(T, 128, 16, rng), _kv4_cache(T, 128, 16, rng)
    o = O.attention_kv4(np.zeros((1, 128), np.float16), K, V, 16, 0.088)
    Vh = O.dequantize_kv(O.unpack_kv(V[0]), V[1], V[2], 16).astype(np.float64)
    assert np.allclose(o[0], Vh.mean(axis=0), rtol=0, atol=1e-12)


def test_attention_kv4_dominant_key_selects_its_value():
    # one key aligned with q and far larger than the rest: o -> V^[t*]
    rng = np.random.default_rng(2)
    T, C = 64, 128
    x = (rng.standard_normal((T, C)) * 0.01).astype(np.float16)
    x[17] = 4.0
    qk, sk, zk = O.quantize_kv_vec(x, 64)
    V = _kv4_cache(T, C, 64, rng)
    q = np.full((1, 128), 1.0, np.float16)
    o = O.attention_kv4(q, (O.pack_kv(qk), sk, zk), V, 64, 1.0)
    Vh = O.dequantize_kv(O.unpack_kv(V[0]), V[1], V[2], 64).astype(np.float64)
    assert np.allclose(o[0], Vh[17], rtol=0, atol=1e-9)


@pytest.mark.gpu
@pytest.mark.parametrize("T,H,G", [(1, 2, 128), (513, 4, 128), (3000, 8, 64), (700, 2, 32), (8192, 32, 128)])
def test_attention_kv4_matches_oracle(T, H, G):
    """GPU dequant-in-attention vs the fp64 oracle over the same KV4 caches:
    |o - o_ref| <= 2^-10 |o_ref| + 2^-12 max|V^| (fp32 dot products, softmax
    and sums in the kernel; one fp16 rounding of o)."""
    import torch
    from paper_2410_12168_b200 import comet
    rng = np.random.default_rng(T + H)
    C = 128 * H
    xk = rng.standard_normal((T, C)).astype(np.float16)
    xv = rng.standard_normal((T, C)).astype(np.float16)
    xk[:, 5] = 0.75  # a constant channel (degenerate group rule)
    q = rng.standard_normal((H, 128)).astype(np.float16)
    dev = torch.device("cuda")
    Kd = comet.comet_quantize_kv(torch.from_numpy(xk).to(dev), G)
    Vd = comet.comet_quantize_kv(torch.from_numpy(xv).to(dev), G)
    o = comet.comet_attention_kv4(torch.from_numpy(q).to(dev), Kd, Vd, G, 128 ** -0.5).float().cpu().numpy()
    K = tuple(t.cpu().numpy() for t in Kd)
    V = tuple(t.cpu().numpy() for t in Vd)
    ref = O.attention_kv4(q, K, V, G, float(np.float32(128 ** -0.5)))
    vmax = np.abs(O.dequantize_kv(O.unpack_kv(V[0]), V[1], V[2], G).astype(np.float64)).max()
    assert np.all(np.abs(o - ref) <= 2.0 ** -10 * np.abs(ref) + 2.0 ** -12 * vmax)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_library_map_equals_oracle(seed):
    rng = np.random.default_rng(seed)
    K = 128 * (seed + 2)
    score = rng.uniform(0.5, 3, K).astype(np.float32)
    score[rng.choice(K, 5 + 40 * seed, replace=False)] *= rng.uniform(10, 100)
    score[rng.choice(K, 4, replace=False)] = score[0]  # ties
    p1, b1, n1 = _lib_map(score)
    p2, b2, n2 = O.fmpq_map(score)
    assert np.array_equal(p1, p2) and np.array_equal(b1, b2) and n1 == n2


def test_library_map_spec_example_and_errors():
    from paper_2410_12168_b200 import comet
    score = np.ones(512, np.float32)
    score[[3, 200, 450]] = [100, 90, 80]
    perm, bits, n = _lib_map(score)
    assert perm[:3].tolist() == [3, 200, 450] and bits.tolist() == [8, 4, 4, 4] and n == 3
    with pytest.raises(comet.CometError):
        _lib_map(np.ones(100, np.float32))  # K % 128
    with pytest.raises(comet.CometError):
        _lib_map(np.ones(128, np.float32), theta=0.5)
    bad = np.ones(128, np.float32)
    bad[5] = np.nan
    with pytest.raises(comet.CometError):
        _lib_map(bad)


# ------------------------------------------------------------- GPU -------
@pytest.mark.gpu
@pytest.mark.parametrize("M,K", [(1, 128), (37, 1024), (512, 4096)])
def test_calib_absmax_bit_exact(M, K):
    import torch
    from paper_2410_12168_b200 import comet
    rng = np.random.default_rng(M + K)
    X = rng.standard_normal((M, K)).astype(np.float16)
    X[:, rng.choice(K, 3, replace=False)] *= np.float16(60)
    X[0, 0] = np.float16(-65504)  # extreme magnitude, negative
    Xd = torch.from_numpy(X).cuda()
    got = comet.comet_calib_absmax(Xd).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), O.calib_absmax(X).view(np.uint32))
    # accumulation over batches == one pass over the concatenation
    X2 = rng.standard_normal((M, K)).astype(np.float16)
    acc = comet.comet_calib_absmax(torch.from_numpy(X2).cuda(), comet.comet_calib_absmax(Xd))
    ref = O.calib_absmax(np.concatenate([X, X2]))
    assert np.array_equal(acc.cpu().numpy().view(np.uint32), ref.view(np.uint32))


@pytest.mark.gpu
def test_calibrated_map_drives_the_w4ax_path():
    """calibrate on the GPU -> map -> pack/quantize/GEMM with that map == oracle."""
    import torch
    import oracle
    from paper_2410_12168_b200 import comet, synth
    p = synth.make_problem(64, 256, 1024, n8=2, seed=7)
    X = torch.from_numpy(p["X"]).cuda()
    score = comet.comet_calib_absmax(X).cpu().numpy()
    perm, bits, n = comet.comet_fmpq_map(score)
    operm, obits, on = O.fmpq_map(score)
    assert np.array_equal(perm, operm) and np.array_equal(bits, obits) and n == on
    assert n >= 32 and (bits == 8).sum() >= 1  # the planted outlier channels are found
    W = torch.from_numpy(p["W"]).cuda()
    pd = torch.from_numpy(perm).cuda()
    Wq, Sw = comet.comet_pack_weight(W, pd, 1024)
    Xq8, Xq4, Sx = comet.comet_quantize_act(X, bits, pd)
    Acc = comet.comet_w4ax_gemm_acc_i32(Xq8, Xq4, Sx, bits, Wq, Sw, 1024)
    oXq8, oXq4, oSx = oracle.quantize_act(p["X"], bits, perm)
    oWq, oSw = oracle.pack_weight(p["W"], 1024, perm)
    r = oracle.w4ax_gemm(oXq8, oXq4, oSx, bits, oWq, oSw, group=1024, want_acc=True)
    assert np.array_equal(Xq8.cpu().numpy(), oXq8) and np.array_equal(Xq4.cpu().numpy(), oXq4)
    assert np.array_equal(Acc.cpu().numpy(), r["acc"])


@pytest.mark.gpu
@pytest.mark.parametrize("T,C,G", [(1, 64, 128), (16, 128, 16), (129, 128, 64), (300, 256, 128),
                                   (1000, 1024, 100), (37, 8, 5), (50, 70, 16), (2048, 4096, 128)])
def test_kv4_bit_exact(T, C, G):
    """vectorised kernels (C % 8 / C % 16 == 0: groups not dividing T, G not a
    multiple of the 8 token lanes, channel tiles of 256 past C) and the
    scalar fallbacks (C = 70; C = 8 dequantizes through the fallback)"""
    import torch
    from paper_2410_12168_b200 import comet
    rng = np.random.default_rng(T * C + G)
    KV = (rng.standard_normal((T, C)) * rng.uniform(0.1, 4, C)).astype(np.float16)
    KV[:, 3] = np.float16(1.75)   # constant channel
    KV[:, 4] = np.float16(-0.5)   # constant negative channel
    KV[:, 5] = 0                  # zero channel
    Kd = torch.from_numpy(KV).cuda()
    Q, s, z = comet.comet_quantize_kv(Kd, G)
    q, os_, oz = O.quantize_kv_vec(KV, G)
    assert np.array_equal(Q.cpu().numpy(), O.pack_kv(q))
    assert np.array_equal(s.cpu().numpy().view(np.uint32), os_.view(np.uint32))
    assert np.array_equal(z.cpu().numpy(), oz)
    Y = comet.comet_dequantize_kv(Q, s, z, G).cpu().numpy()
    assert np.array_equal(Y.view(np.uint16), O.dequantize_kv(q, os_, oz, G).view(np.uint16))
