"""Pre-expanded weights (a4 done offline, comet_expand_weight) and the GEMM
that consumes them (comet_w4ax_gemm_ex): We must equal 16 x the oracle's
unpacked INT4 weights bit for bit, and Y must be identical to
comet_w4ax_gemm's (same integer block sums, same promotion order) and within
the tolerance of the oracle."""
import numpy as np
import pytest

import oracle
from paper_2410_12168_b200 import synth


@pytest.mark.gpu
@pytest.mark.parametrize("N,K,group", [(128, 128, 128), (384, 1024, "K"), (11008 // 128 * 128, 512, 128)])
def test_expand_weight_bit_exact(N, K, group):
    import torch
    from paper_2410_12168_b200 import comet

    rng = np.random.default_rng(N + K)
    W = (rng.standard_normal((N, K)) * 0.05).astype(np.float16)
    perm = rng.permutation(K).astype(np.int32)
    dev = torch.device("cuda")
    g = K if group == "K" else 128
    Wq, Sw = comet.comet_pack_weight(torch.from_numpy(W).to(dev), torch.from_numpy(perm).to(dev), g)
    We = comet.comet_expand_weight(Wq).cpu().numpy()
    Wq_o, _ = oracle.pack_weight(W, g, perm)
    ref = oracle.unpack_int4(Wq_o.reshape(-1), N * K).reshape(N, K).astype(np.int16) * 16
    assert np.array_equal(We.astype(np.int16), ref)


@pytest.mark.gpu
@pytest.mark.parametrize("M,N,K,group", [(300, 384, 1024, 128), (257, 640, 2048, "K"), (4096, 4096, 4096, "K"),
                                          (16, 256, 512, 128)])
def test_gemm_ex_identical_to_gemm(M, N, K, group):
    import torch
    from paper_2410_12168_b200 import comet

    p = synth.make_problem(M, N, K, n8=max(1, K // 128 // 8), seed=M + N)
    dev = torch.device("cuda")
    g = K if group == "K" else 128
    X = torch.from_numpy(p["X"]).to(dev)
    perm = torch.from_numpy(p["perm"]).to(dev)
    Xq8, Xq4, Sx = comet.comet_quantize_act(X, p["bits"], perm)
    Wq, Sw = comet.comet_pack_weight(torch.from_numpy(p["W"]).to(dev), perm, g)
    We = comet.comet_expand_weight(Wq)
    ws = comet.new_workspace(comet.comet_w4ax_gemm_workspace_bytes(M, N, K), dev)
    Y0 = comet.comet_w4ax_gemm(Xq8, Xq4, Sx, p["bits"], Wq, Sw, g, workspace=ws)
    Y1 = comet.comet_w4ax_gemm_ex(Xq8, Xq4, Sx, p["bits"], Wq, We, Sw, g, workspace=ws)
    assert torch.equal(Y0.view(torch.int16), Y1.view(torch.int16))
    rows = np.arange(M) if M <= 512 else np.r_[0, M - 1, np.random.default_rng(1).choice(M, 30, replace=False)]
    Wq_o, Sw_o = oracle.pack_weight(p["W"], g, p["perm"])
    r8, r4, rs = oracle.quantize_act(p["X"][rows], p["bits"], p["perm"])
    ref = oracle.w4ax_gemm(r8, r4, rs, p["bits"], Wq_o, Sw_o, g)["y"].astype(np.float32)
    y = Y1.float().cpu().numpy()[rows]
    assert np.all(np.abs(y - ref) <= np.maximum(2.0 ** -10 * np.abs(ref), 1e-3))
