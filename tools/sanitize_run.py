"""Small runs of every GEMM path for compute-sanitizer (tools/gpu_sanitize.sh):
C1 tiny (decode kernel), a ragged prefill (CTA-pair kernel + token prep), the
linear entry (fused quantizer), the INT32 debug entry, the thread-per-item
quantizer (M >= 512, with / without the permutation, packed and e4m3 output)
and the fused all-gather entries (two destinations)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_12168_b200 import comet, synth  # noqa: E402

for (M, N, K, n8) in [(16, 256, 512, 1), (300, 640, 1024, 2), (600, 384, 2048, 2)]:
    p = synth.make_problem(M, N, K, n8=n8, seed=1, mask="scattered")
    X, W, perm = (torch.from_numpy(p[k]).cuda() for k in ("X", "W", "perm"))
    bits = comet.BlockBits(p["bits"])
    for g in (128, K):
        Wq, Sw = comet.comet_pack_weight(W, perm, g)
        Xq8, Xq4, Sx = comet.comet_quantize_act(X, bits, perm)
        ws = comet.new_workspace(comet.comet_w4ax_gemm_workspace_bytes(M, N, K), X.device)
        comet.comet_w4ax_gemm(Xq8, Xq4, Sx, bits, Wq, Sw, g, workspace=ws)
        comet.comet_w4ax_gemm_acc_i32(Xq8, Xq4, Sx, bits, Wq, Sw, g)
        scratch = comet.new_workspace(comet.comet_w4ax_linear_scratch_bytes(M, N, K, bits), X.device)
        comet.comet_w4ax_linear(X, bits, Wq, Sw, perm=perm, group=g, scratch=scratch)
        comet.comet_quantize_act(X, bits, None)
        dests = [torch.empty((M, 2 * N), dtype=torch.float16, device=X.device) for _ in range(2)]
        comet.comet_w4ax_linear_allgather(X, bits, Wq, Sw, dests, 2 * N, N, perm=perm, group=g, scratch=scratch)
        comet.comet_w4ax_gemm_allgather(Xq8, Xq4, Sx, bits, Wq, Sw, dests, 2 * N, 0, g, workspace=ws)
torch.cuda.synchronize()
print("sanitize run done")
