"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle (-m gpu).

Bars (BJ north_star):
  * packed planes Xq8/Xq4, scales Sx, packed weights Wq and Sw: bit-exact;
  * per-block INT32 accumulators (comet_w4ax_gemm_acc_i32): bit-exact;
  * Y fp16: |y - y_ref| <= max(2^-10 |y_ref|, 1e-3) elementwise.
Inputs come from paper_2410_12168_b200.synth (seeded); expected values only
from oracle/.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2410_12168_b200 import comet, synth

pytestmark = pytest.mark.gpu

REL, ABS = 2.0 ** -10, 1e-3


def to_dev(a):
    return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()


def gpu_path(p, group, want_acc=False, planes_only=False):
    X, W = to_dev(p["X"]), to_dev(p["W"])
    perm = to_dev(p["perm"])
    bits = comet.BlockBits(p["bits"])
    Wq, Sw = comet.comet_pack_weight(W, perm, group)
    Xq8, Xq4, Sx = comet.comet_quantize_act(X, bits, perm)
    out = {"Wq": Wq, "Sw": Sw, "Xq8": Xq8, "Xq4": Xq4, "Sx": Sx}
    if not planes_only:
        M, N, K = X.shape[0], W.shape[0], X.shape[1]
        ws = comet.new_workspace(comet.comet_w4ax_gemm_workspace_bytes(M, N, K), X.device)
        out["Y"] = comet.comet_w4ax_gemm(Xq8, Xq4, Sx, bits, Wq, Sw, group, workspace=ws)
        if want_acc:
            out["Acc"] = comet.comet_w4ax_gemm_acc_i32(Xq8, Xq4, Sx, bits, Wq, Sw, group)
    torch.cuda.synchronize()
    res = {k: v.cpu().numpy() for k, v in out.items()}
    N, K = p["W"].shape
    res["Wq"] = comet.wq_tiled_to_rowmajor(res["Wq"], N, K)  # layout only
    return res


def oracle_path(p, group, rows=None, want_acc=False):
    Xq8, Xq4, Sx = oracle.quantize_act(p["X"], p["bits"], p["perm"])
    Wq, Sw = oracle.pack_weight(p["W"], group, p["perm"])
    r = oracle.w4ax_gemm(Xq8, Xq4, Sx, p["bits"], Wq, Sw, group=group, rows=rows, want_acc=want_acc, want_y64=True)
    return {"Xq8": Xq8, "Xq4": Xq4, "Sx": Sx, "Wq": Wq, "Sw": Sw, **r}


def assert_planes_equal(g, o):
    for k in ("Xq8", "Xq4", "Wq"):
        assert g[k].shape == o[k].shape, k
        assert np.array_equal(g[k].view(np.uint8), o[k].view(np.uint8)), k
    for k in ("Sx", "Sw"):
        assert np.array_equal(g[k].view(np.uint32), o[k].view(np.uint32)), k


def assert_y_close(y_gpu, y_ref16, y64):
    ref = y_ref16.astype(np.float64)
    yg = y_gpu.astype(np.float64)
    tol = np.maximum(REL * np.abs(ref), ABS)
    bad = np.abs(yg - ref) > tol
    assert not bad.any(), f"{bad.sum()} mismatches, worst {np.abs(yg - ref)[bad].max()}"
    assert np.all(np.abs(yg - y64) <= np.maximum(REL * np.abs(y64), ABS) + np.abs(ref - y64))


# ------------------------------------------------------------- C1 tiny ----
C1_MASKS = [[8, 4, 4, 4], [4, 4, 8, 4], [4, 4, 4, 4], [8, 8, 8, 8]]


@pytest.mark.parametrize("mask", C1_MASKS)
@pytest.mark.parametrize("group", [128, 512])
@pytest.mark.parametrize("seed", [0, 1])
def test_c1_tiny_full_parity(mask, group, seed):
    """BJ configs[0]: M=16 N=256 K=512, block 128, one INT8 outlier block."""
    n8 = sum(1 for b in mask if b == 8)
    p = synth.make_problem(16, 256, 512, n8=n8, seed=seed, mask=mask)
    g = gpu_path(p, group, want_acc=True)
    o = oracle_path(p, group, want_acc=True)
    assert_planes_equal(g, o)
    assert np.array_equal(g["Acc"], o["acc"])
    assert_y_close(g["Y"], o["y"], o["y64"])


@pytest.mark.parametrize("group", [128, 1024])
@pytest.mark.parametrize("M", [1, 3, 5, 13, 16, 17, 31, 33, 64, 65, 100, 128, 129, 255, 256, 300, 520])
def test_ragged_m_all_tile_widths(M, group):
    """Every kernel specialisation (decode BN 16/32/64/128, CTA-pair prefill
    for M > 128), ragged token tails, N = 384 (a half-populated pair tile),
    group-128 and per-channel weight scales."""
    p = synth.make_problem(M, 384, 1024, n8=1, seed=100 + M, mask="scattered")
    g = gpu_path(p, group, want_acc=True)
    o = oracle_path(p, group, want_acc=True)
    assert_planes_equal(g, o)
    assert np.array_equal(g["Acc"], o["acc"])
    assert_y_close(g["Y"], o["y"], o["y64"])


@pytest.mark.parametrize("N", [128, 256, 512, 640, 768])
@pytest.mark.parametrize("group", [128, 1024])
def test_prefill_pair_tile_edges(N, group):
    """Prefill pair tiles are 192 weight channels (96 per CTA): N % 192 in
    {0, 64, 128} gives tiles whose second CTA holds a partial slab (v < 96),
    straddles a 128-row slab of the tiled weight layout, or has no rows."""
    p = synth.make_problem(300, N, 1024, n8=2, seed=500 + N, mask="scattered")
    g = gpu_path(p, group, want_acc=True)
    o = oracle_path(p, group, want_acc=True)
    assert_planes_equal(g, o)
    assert np.array_equal(g["Acc"], o["acc"])
    assert_y_close(g["Y"], o["y"], o["y64"])


@pytest.mark.parametrize("M,N,K", [(1, 4096, 4096), (16, 1024, 4096), (8, 512, 8192), (128, 256, 2048)])
def test_split_k_decode_shapes(M, N, K):
    """Few tiles -> split-K with the deterministic last-CTA fixup (a7)."""
    assert comet.comet_w4ax_gemm_workspace_bytes(M, N, K) > 0
    p = synth.make_problem(M, N, K, n8=K // 128 // 10, seed=7)
    g = gpu_path(p, 128)
    o = oracle_path(p, 128)
    assert_planes_equal(g, o)
    assert_y_close(g["Y"], o["y"], o["y64"])


def test_no_permutation_and_outliers_unclustered():
    p = synth.make_problem(48, 256, 1024, n8=2, seed=3, with_perm=False)
    g = gpu_path(p, 128, want_acc=True)
    o = oracle_path(p, 128, want_acc=True)
    assert_planes_equal(g, o)
    assert np.array_equal(g["Acc"], o["acc"])
    assert_y_close(g["Y"], o["y"], o["y64"])


def test_permutation_equivalence_on_gpu():
    """P8: fused gather == pre-permuted input, bit-identical planes and Y."""
    p = synth.make_problem(64, 256, 1024, n8=1, seed=5)
    q = dict(p)
    q["X"] = np.ascontiguousarray(p["X"][:, p["perm"]])
    q["W"] = np.ascontiguousarray(p["W"][:, p["perm"]])
    q["perm"] = None
    a, b = gpu_path(p, 128), gpu_path(q, 128)
    for k in a:
        assert np.array_equal(a[k].view(np.uint8), b[k].view(np.uint8)), k


def test_power_of_two_scales_bit_exact():
    """P11: exact scales and products -> GPU fp16 Y bit-equal to the oracle."""
    rng = np.random.default_rng(12)
    M, N, K = 32, 256, 512
    X = rng.integers(-7, 8, (M, K)).astype(np.float64)
    X[:, :128] = rng.integers(-127, 128, (M, 128)) * 0.25
    X[:, 0], X[:, 128], X[:, 256], X[:, 384] = 127 * 0.25, 7, -7, 7
    W = rng.integers(-7, 8, (N, K)).astype(np.float64) * 0.5
    W[:, 0::128] = 3.5
    p = {"X": X.astype(np.float16), "W": W.astype(np.float16), "perm": None, "bits": np.array([8, 4, 4, 4], np.uint8)}
    g = gpu_path(p, 128)
    o = oracle_path(p, 128)
    assert np.array_equal(o["y64"], X @ W.T)
    assert np.array_equal(g["Y"].view(np.uint16), o["y"].view(np.uint16))


def test_zero_padded_brute_force_8x8x64():
    """P9 on the GPU: real 8x8x64 problem zero-padded to the ABI shape
    (M=8, N=128, K=128) equals the k=64 oracle in the 8x8 corner."""
    rng = np.random.default_rng(10)
    X = (rng.standard_normal((8, 64)) * 2).astype(np.float16)
    W = (rng.standard_normal((8, 64)) / 8).astype(np.float16)
    b64 = np.array([4], np.uint8)
    r64 = oracle.w4ax_gemm(*oracle.quantize_act(X, b64, None, k=64), b64, *oracle.pack_weight(W, 64), group=64, k=64,
                           want_y64=True)
    Xp = np.zeros((8, 128), np.float16)
    Xp[:, :64] = X
    Wp = np.zeros((128, 128), np.float16)
    Wp[:8, :64] = W
    g = gpu_path({"X": Xp, "W": Wp, "perm": None, "bits": np.array([4], np.uint8)}, 128)
    assert_y_close(g["Y"][:, :8], r64["y64"].astype(np.float16), r64["y64"])
    assert not g["Y"][:, 8:].any()


def test_zero_blocks_and_zero_rows():
    """A-7: all-zero blocks get s = 1 and q = 0; zero weight rows give Y = 0."""
    p = synth.make_problem(20, 256, 512, n8=1, seed=4)
    p["X"][3, :] = 0
    p["X"][5, 128:256] = 0
    p["W"][7, :] = 0
    g = gpu_path(p, 128, want_acc=True)
    o = oracle_path(p, 128, want_acc=True)
    assert_planes_equal(g, o)
    assert np.array_equal(g["Acc"], o["acc"])
    assert not g["Y"][3].any() and not g["Y"][:, 7].any()


def test_determinism():
    p = synth.make_problem(16, 2048, 4096, n8=3, seed=8)
    a, b = gpu_path(p, 128), gpu_path(p, 128)
    assert np.array_equal(a["Y"].view(np.uint16), b["Y"].view(np.uint16))


def test_fp16_extremes_quantize_bit_exact():
    """Adversarial activations: +-65504, subnormals, -0, exact ties."""
    rng = np.random.default_rng(2)
    X = rng.standard_normal((8, 512)).astype(np.float16)
    X[0, :8] = [65504, -65504, 6e-8, -6e-8, -0.0, 0.5, 1.5, 2.5]
    X[1, :128] = np.float16(6e-8) * rng.integers(-20, 20, 128)  # subnormal block
    X[2, 128:136] = [7, 3.5, -3.5, 1.5, 0.5, -0.5, 2.5, -2.5]    # ties at r == 1
    X[3, 256:384] = 0
    p = {"X": X, "W": np.zeros((128, 512), np.float16), "perm": None, "bits": np.array([4, 4, 8, 4], np.uint8)}
    g = gpu_path(p, 128, planes_only=True)
    o = oracle_path(p, 128)
    for k in ("Xq8", "Xq4", "Sx"):
        assert np.array_equal(g[k].view(np.uint8), o[k].view(np.uint8)), k


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
def test_quantize_every_block_absmax_bit_exact(dtype):
    """The row-staged quantizer derives s = a/qmax and r = qmax/a from a table
    of the 1024 mantissas scaled by the exponent of a: sweep every positive
    fp16 value (and a bf16 exponent range) as a block absmax, INT4 and INT8
    blocks, planes and Sx bit-exact against the oracle's IEEE divisions."""
    import importlib
    rng = np.random.default_rng(11)
    K = 1024
    bits = np.array([4, 8, 4, 4, 8, 4, 4, 4], np.uint8)
    if dtype == "fp16":
        amax = np.arange(1, 0x7C00, dtype=np.uint16).view(np.float16).astype(np.float32)  # every finite positive fp16
    else:
        e = rng.integers(-100, 100, size=40000)
        mant = rng.integers(0, 128, size=40000)
        amax = ((1.0 + mant / 128.0) * 2.0 ** e).astype(np.float32)  # exact bf16 values
    nitems = len(amax)
    M = -(-nitems // 8)
    a = np.resize(amax, M * 8).reshape(M, 8)
    frac = rng.uniform(-1.0, 1.0, size=(M, 8, 128)).astype(np.float32)
    X32 = frac * a[:, :, None]
    X32[:, :, 0] = a  # the block absmax, exactly
    X32 = X32.reshape(M, K)
    bitsb = comet.BlockBits(bits)
    if dtype == "fp16":
        X = X32.astype(np.float16)
        g8, g4, gs = comet.comet_quantize_act(to_dev(X), bitsb, None)
        o8, o4, os_ = oracle.quantize_act(X, bits, None)
    else:
        O = importlib.import_module("oracle.fmpq_aux")
        b16 = (X32.view(np.uint32) >> 16).astype(np.uint16)  # truncation: keeps the exact bf16 absmax
        g8, g4, gs = comet.comet_quantize_act_bf16(to_dev(b16.view(np.int16)).view(torch.bfloat16), bitsb, None)
        o8, o4, os_ = O.quantize_act_bf16(b16, bits)
    torch.cuda.synchronize()
    assert np.array_equal(g8.cpu().numpy(), o8) and np.array_equal(g4.cpu().numpy(), o4)
    assert np.array_equal(gs.cpu().numpy().view(np.uint32), os_.view(np.uint32))


def test_quantize_random_rows_bit_exact_large():
    """10^5-ish random rows across scales: planes and scales bit-exact."""
    rng = np.random.default_rng(77)
    M, K = 4096, 1024
    X = (rng.standard_normal((M, K)) * 10.0 ** rng.uniform(-4, 4, (M, 1))).astype(np.float16)
    bits = synth.block_bits_for(K, 2, "scattered")
    p = {"X": X, "W": np.zeros((128, K), np.float16), "perm": None, "bits": bits}
    g = gpu_path(p, 128, planes_only=True)
    Xq8, Xq4, Sx = oracle.quantize_act(X, bits)
    assert np.array_equal(g["Xq8"], Xq8) and np.array_equal(g["Xq4"], Xq4)
    assert np.array_equal(g["Sx"].view(np.uint32), Sx.view(np.uint32))


# ------------------------------------------------- full-size (sampled) ----
@pytest.mark.parametrize("M,N,K,n8,group", [(4096, 11008, 4096, 3, 128), (4096, 4096, 4096, 3, 4096),
                                             (16, 57344, 8192, 6, 128), (2048, 8192, 28672, 22, 128)])
def test_full_size_sampled_rows(M, N, K, n8, group):
    """BJ configs at full size in the launch configuration bench.py times:
    planes/scales bit-exact over ALL rows; INT32 + Y on a 64-row sample."""
    p = synth.make_problem(M, N, K, n8=n8, seed=300)
    g = gpu_path(p, group)
    Xq8, Xq4, Sx = oracle.quantize_act(p["X"], p["bits"], p["perm"])
    assert np.array_equal(g["Xq8"], Xq8) and np.array_equal(g["Xq4"], Xq4)
    assert np.array_equal(g["Sx"].view(np.uint32), Sx.view(np.uint32))
    Wq, Sw = oracle.pack_weight(p["W"], group, p["perm"])
    assert np.array_equal(g["Wq"], Wq) and np.array_equal(g["Sw"].view(np.uint32), Sw.view(np.uint32))
    rows = synth.sample_rows(M, 64 if M > 64 else M)
    r = oracle.w4ax_gemm(Xq8, Xq4, Sx, p["bits"], Wq, Sw, group=group, rows=rows, want_y64=True)
    assert_y_close(g["Y"][rows], r["y"], r["y64"])


def test_linear_entry_with_host_buffers():
    """comet_w4ax_linear: host X in, host Y out, same result as the device path."""
    p = synth.make_problem(100, 512, 1024, n8=1, seed=9)
    g = gpu_path(p, 128)
    W = to_dev(p["W"])
    perm = to_dev(p["perm"])
    bits = comet.BlockBits(p["bits"])
    Wq, Sw = comet.comet_pack_weight(W, perm, 128)
    Xh = torch.from_numpy(p["X"]).pin_memory()
    Yh = torch.empty((100, 512), dtype=torch.float16).pin_memory()
    scratch = comet.new_workspace(comet.comet_w4ax_linear_scratch_bytes(100, 512, 1024, bits), W.device)
    comet.comet_w4ax_linear(Xh, bits, Wq, Sw, perm=perm, out=Yh, scratch=scratch)
    assert np.array_equal(Yh.numpy().view(np.uint16), g["Y"].view(np.uint16))


@pytest.mark.parametrize("M,K,n8,group", [(301, 1024, 2, 128), (517, 1024, 2, 1024), (300, 1152, 3, 1152),
                                           (260, 2176, 5, 128)])
def test_linear_prefill_fused_quantizer(M, K, n8, group):
    """comet_w4ax_linear at prefill sizes: the quantizer writes the GEMM's e4m3
    token operand and corrections directly (no packed plane, no prep kernel);
    Y must be bit-identical to the two-call path (same tcgen05 arithmetic),
    ragged M (ldsx padding rows), scattered INT8 blocks (the two half-warps of
    a warp may hold an INT8 and an INT4 block), odd block counts (the last
    half-warp idles), both scale kinds."""
    p = synth.make_problem(M, 640, K, n8=n8, seed=31 + M, mask="scattered")
    ref = gpu_path(p, group)["Y"]
    W, perm, X = to_dev(p["W"]), to_dev(p["perm"]), to_dev(p["X"])
    bits = comet.BlockBits(p["bits"])
    Wq, Sw = comet.comet_pack_weight(W, perm, group)
    scratch = comet.new_workspace(comet.comet_w4ax_linear_scratch_bytes(M, 640, K, bits), W.device)
    Y = comet.comet_w4ax_linear(X, bits, Wq, Sw, perm=perm, group=group, scratch=scratch)
    torch.cuda.synchronize()
    assert np.array_equal(Y.cpu().numpy().view(np.uint16), ref.view(np.uint16))


def test_linear_host_calls_overlap_without_sync():
    """Consecutive host-buffer calls (sync=False) overlap their copies: the
    input copies of a call start after the previous call's compute, not its
    output copies.  Same scratch reused by calls of different shapes (the
    second call's staged X overlaps the first call's staged Y, so that case
    must wait for the first call's output copies), a separate scratch, and a
    device-buffer call in between; every Y must equal its device-buffer
    result after one synchronize."""
    cases = [(2600, 640, 1024, 2, 41), (2300, 1024, 2048, 3, 42), (2100, 512, 1152, 3, 43)]
    shared = None
    jobs = []
    for i, (M, N, K, n8, seed) in enumerate(cases):
        p = synth.make_problem(M, N, K, n8=n8, seed=seed, mask="scattered")
        W, perm = to_dev(p["W"]), to_dev(p["perm"])
        bits = comet.BlockBits(p["bits"])
        Wq, Sw = comet.comet_pack_weight(W, perm, 128)
        need = comet.comet_w4ax_linear_scratch_bytes(M, N, K, bits)
        own = comet.new_workspace(need, W.device)
        ref = comet.comet_w4ax_linear(to_dev(p["X"]), bits, Wq, Sw, perm=perm, scratch=own).cpu().numpy()
        jobs.append((p, bits, Wq, Sw, perm, M, N, own, ref))
    need = max(comet.comet_w4ax_linear_scratch_bytes(j[5], j[6], j[0]["X"].shape[1], j[1]) for j in jobs)
    shared = comet.new_workspace(need, jobs[0][2].device)
    torch.cuda.synchronize()
    outs = []
    for i, (p, bits, Wq, Sw, perm, M, N, own, ref) in enumerate(jobs):
        Xh = torch.from_numpy(p["X"]).pin_memory()
        Yh = torch.full((M, N), float("nan"), dtype=torch.float16).pin_memory()
        scratch = own if i == 1 else shared
        comet.comet_w4ax_linear(Xh, bits, Wq, Sw, perm=perm, out=Yh, scratch=scratch, sync=False)
        if i == 1:  # a device-buffer call on the shared scratch between host calls
            pd = jobs[0]
            dev_y = comet.comet_w4ax_linear(to_dev(pd[0]["X"]), pd[1], pd[2], pd[3], perm=pd[4], scratch=shared)
            outs.append((dev_y, pd[8]))
        outs.append((Yh, ref))
    torch.cuda.synchronize()
    for Y, ref in outs:
        assert np.array_equal(Y.cpu().numpy().view(np.uint16), ref.view(np.uint16))


def test_linear_host_buffers_pipelined_chunks():
    """Host X and Y at M >= 2048: the call pipelines row chunks (H2D / layer /
    D2H on internal copy streams); Y must equal the device-buffer call."""
    M, N, K = 2600, 640, 1024
    p = synth.make_problem(M, N, K, n8=2, seed=41, mask="scattered")
    W, perm = to_dev(p["W"]), to_dev(p["perm"])
    bits = comet.BlockBits(p["bits"])
    Wq, Sw = comet.comet_pack_weight(W, perm, 128)
    scratch = comet.new_workspace(comet.comet_w4ax_linear_scratch_bytes(M, N, K, bits), W.device)
    Yd = comet.comet_w4ax_linear(to_dev(p["X"]), bits, Wq, Sw, perm=perm, scratch=scratch)
    torch.cuda.synchronize()
    Xh = torch.from_numpy(p["X"]).pin_memory()
    Yh = torch.empty((M, N), dtype=torch.float16).pin_memory()
    comet.comet_w4ax_linear(Xh, bits, Wq, Sw, perm=perm, out=Yh, scratch=scratch)
    assert np.array_equal(Yh.numpy().view(np.uint16), Yd.cpu().numpy().view(np.uint16))


def test_linear_prefill_then_decode_same_scratch():
    """a prefill call (no GEMM workspace) must not overwrite the
    stream-K tile counters a later decode call on the same scratch uses."""
    bits_np = synth.block_bits_for(4096, 3)
    bits = comet.BlockBits(bits_np)
    pre = synth.make_problem(4096, 4096, 4096, n8=3, seed=21)
    dec = synth.make_problem(16, 4096, 4096, n8=3, seed=22)
    dec["perm"], dec["W"] = pre["perm"], pre["W"]  # one layer, two calls
    W, perm = to_dev(pre["W"]), to_dev(pre["perm"])
    Wq, Sw = comet.comet_pack_weight(W, perm, 128)
    need = max(comet.comet_w4ax_linear_scratch_bytes(m, 4096, 4096, bits) for m in (4096, 16))
    scratch = torch.full((need,), 0, dtype=torch.uint8, device=W.device)
    for p in (pre, dec, dec):
        X = to_dev(p["X"])
        Y = comet.comet_w4ax_linear(X, bits, Wq, Sw, perm=perm, scratch=scratch)
        torch.cuda.synchronize()
        ref = gpu_path(p, 128)["Y"]
        assert np.array_equal(Y.cpu().numpy().view(np.uint16), ref.view(np.uint16))


def acc_sampled(p, group, rows):
    """GPU per-block INT32 accumulators of the full problem, sampled rows."""
    X, W, perm = to_dev(p["X"]), to_dev(p["W"]), to_dev(p["perm"])
    bits = comet.BlockBits(p["bits"])
    Wq, Sw = comet.comet_pack_weight(W, perm, group)
    Xq8, Xq4, Sx = comet.comet_quantize_act(X, bits, perm)
    Acc = comet.comet_w4ax_gemm_acc_i32(Xq8, Xq4, Sx, bits, Wq, Sw, group)
    out = Acc[:, torch.from_numpy(rows).long().cuda(), :].cpu().numpy()
    del Acc
    torch.cuda.empty_cache()
    return out


@pytest.mark.parametrize("M,N,K,n8,group", [(4096, 11008, 4096, 3, 128), (2048, 8192, 28672, 22, 128),
                                             (16, 57344, 8192, 6, 128), (8192, 6144, 4096, 3, 4096)])
def test_full_size_acc_i32_sampled_rows(M, N, K, n8, group):
    """INT32 bit-exactness in the launch configurations the bench runs:
    multi-tile persistent prefill loops (ring phases flip across tiles) and
    multi-unit stream-K decode; 64 sampled rows (first, last, seeded random)."""
    p = synth.make_problem(M, N, K, n8=n8, seed=310)
    rows = synth.sample_rows(M, 64 if M > 64 else M)
    g = acc_sampled(p, group, rows)
    Xq8, Xq4, Sx = oracle.quantize_act(p["X"], p["bits"], p["perm"])
    Wq, Sw = oracle.pack_weight(p["W"], group, p["perm"])
    r = oracle.w4ax_gemm(Xq8, Xq4, Sx, p["bits"], Wq, Sw, group=group, rows=rows, want_acc=True)
    assert g.shape == r["acc"].shape
    assert np.array_equal(g, r["acc"])


def pow2_problem(M, N, K, n8, seed):
    """P11 inputs: every (row, block) absmax is qmax * 2^e (INT4 blocks 7 * 1,
    INT8 blocks 127 * 0.25) and every weight group's absmax is 7 * 0.5, all
    values on those lattices: every scale, product and partial sum is exact."""
    rng = np.random.default_rng(seed)
    bits = synth.block_bits_for(K, n8, "scattered")
    X = rng.integers(-7, 8, (M, K)).astype(np.float64)
    sgn = lambda shape: np.where(rng.integers(0, 2, shape) == 1, 1.0, -1.0)
    for b in range(K // 128):
        if bits[b] == 8:
            X[:, b * 128:(b + 1) * 128] = rng.integers(-127, 128, (M, 128)) * 0.25
            X[:, b * 128] = 127 * 0.25 * sgn(M)
        else:
            X[:, b * 128] = 7 * sgn(M)
    W = rng.integers(-7, 8, (N, K)).astype(np.float64) * 0.5
    W[:, 0::128] = 3.5 * sgn((N, K // 128))
    return {"X": X.astype(np.float16), "W": W.astype(np.float16), "perm": None, "bits": bits}


@pytest.mark.parametrize("M,group", [(300, 128), (300, 4096), (4096, 128), (4096, 4096)])
def test_power_of_two_scales_bit_exact_prefill(M, group):
    """P11 on the prefill kernel (M > 128) with N = 14336 >= 74 clusters x 192
    (every cluster runs tiles; M = 4096 loops several tiles per cluster):
    fp16 Y bit-equal to the oracle on 64 sampled rows."""
    N, K = 14336, 4096
    p = pow2_problem(M, N, K, 3, seed=40 + M)
    g = gpu_path(p, group)
    rows = synth.sample_rows(M, 64)
    Xq8, Xq4, Sx = oracle.quantize_act(p["X"], p["bits"], None)
    Wq, Sw = oracle.pack_weight(p["W"], group, None)
    r = oracle.w4ax_gemm(Xq8, Xq4, Sx, p["bits"], Wq, Sw, group=group, rows=rows, want_y64=True)
    assert np.array_equal(r["y64"], p["X"][rows].astype(np.float64) @ p["W"].astype(np.float64).T)
    assert np.array_equal(g["Y"][rows].view(np.uint16), r["y"].view(np.uint16))


@pytest.mark.parametrize("M", [65, 100, 128])
def test_kernel_choice_band_both_kernels(M):
    """64 < M <= 128 with per-channel weight scales runs the CTA-pair prefill
    kernel (faster there, profiles/mband_sweep_r2.txt); the decode kernel's
    BN = 128 per-channel specialisation stays checked by forcing it through
    the tools-only comet_debug_set_prefill_min_m hook."""
    import ctypes
    L = comet.lib()
    L.comet_debug_set_prefill_min_m.argtypes = [ctypes.c_int]
    p = synth.make_problem(M, 640, 2048, n8=2, seed=900 + M, mask="scattered")
    o = oracle_path(p, 2048, want_acc=True)
    try:
        for force in (0, 1000):
            L.comet_debug_set_prefill_min_m(force)
            g = gpu_path(p, 2048, want_acc=True)
            assert_planes_equal(g, o)
            assert np.array_equal(g["Acc"], o["acc"])
            assert_y_close(g["Y"], o["y"], o["y64"])
    finally:
        L.comet_debug_set_prefill_min_m(0)
