"""Decode vs prefill kernel in the M = 64..128 band (tools only): the same GEMM
timed with the product kernel choice and with the other kernel forced via
comet_debug_set_prefill_min_m.
    python tools/mband_sweep.py"""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2410_12168_b200 import comet, synth

L = comet.lib()
L.comet_debug_set_prefill_min_m.argtypes = [ctypes.c_int]


def time_gemm(M, N, K, n8, group, reps=20):
    dev = torch.device("cuda")
    bits = comet.BlockBits(synth.block_bits_for(K, n8))
    X = torch.randn(M, K, device=dev).half()
    W = (torch.randn(N, K, device=dev) / K ** 0.5).half()
    Wq, Sw = comet.comet_pack_weight(W, None, group)
    Xq8, Xq4, Sx = comet.comet_quantize_act(X, bits, None)
    ws = comet.new_workspace(max(comet.comet_w4ax_gemm_workspace_bytes(M, N, K), 1), dev)
    Y = torch.empty(M, N, dtype=torch.float16, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ts = []
    for i in range(reps + 3):
        flush.fill_(1)
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        comet.comet_w4ax_gemm(Xq8, Xq4, Sx, bits, Wq, Sw, group, out=Y, workspace=ws)
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    return float(np.median(ts)) * 1e3


if __name__ == "__main__":
    for (N, K, n8) in [(57344, 8192, 6), (28672, 4096, 3), (4096, 14336, 11)]:
        for g in ("channel", 128):
            grp = K if g == "channel" else 128
            for M in (48, 64, 80, 96, 112, 128, 144):
                L.comet_debug_set_prefill_min_m(1000000)  # decode kernel
                td = time_gemm(M, N, K, n8, grp) if M <= 128 else None
                L.comet_debug_set_prefill_min_m(1)        # prefill kernel
                tp = time_gemm(M, N, K, n8, grp)
                L.comet_debug_set_prefill_min_m(0)
                print(json.dumps({"N": N, "K": K, "M": M, "group": g, "decode_us": td, "prefill_us": tp}))
