"""Time the FMPQ side kernels with CUDA events, L2 flushed.

    python tools/aux_bench.py   -> one JSON line per kernel (GB/s vs measured HBM peak)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2410_12168_b200 import comet

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def peak():
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(d.get("hbm_gbs") or d.get("hbm_copy_gbs"))
    except Exception:
        return 6650.0


def timed(fn, reps=20):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for i in range(reps + 3):
        flush.fill_(1)
        torch.cuda._sleep(1_000_000)
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); fn(); b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b) * 1e-3)
    return float(np.median(ts))


def main():
    pk = peak()
    out = []
    # f2: calibration absmax over a 4096-token batch of a K=8192 activation
    X = torch.randn(4096, 8192, device="cuda").half()
    acc = torch.zeros(8192, device="cuda")
    t = timed(lambda: comet.comet_calib_absmax(X, acc))
    out.append({"kernel": "calib_absmax", "shape": [4096, 8192], "us": t * 1e6, "GBs": X.numel() * 2 / t / 1e9})
    # f3: KV4 quantize-on-append of a prefill chunk: 8192 tokens x (8 kv heads x 128 dims), group 128
    KV = torch.randn(8192, 1024, device="cuda").half()
    t = timed(lambda: comet.comet_quantize_kv(KV, 128))
    byts = KV.numel() * 2 + KV.numel() // 2 + 8192 // 128 * 1024 * 5
    out.append({"kernel": "kv4_quantize", "shape": [8192, 1024, 128], "us": t * 1e6, "GBs": byts / t / 1e9})
    Q, s, z = comet.comet_quantize_kv(KV, 128)
    t = timed(lambda: comet.comet_dequantize_kv(Q, s, z, 128))
    byts = KV.numel() // 2 + KV.numel() * 2 + 8192 // 128 * 1024 * 5
    out.append({"kernel": "kv4_dequantize", "shape": [8192, 1024, 128], "us": t * 1e6, "GBs": byts / t / 1e9})
    # the same at a size where the fixed launch cost (~5 us per event-timed kernel) stops mattering:
    # 131072 tokens (a 32k context x 4 sequences) x 1024
    KVb = torch.randn(131072, 1024, device="cuda").half()
    t = timed(lambda: comet.comet_quantize_kv(KVb, 128))
    byts = KVb.numel() * 2 + KVb.numel() // 2 + 131072 // 128 * 1024 * 5
    out.append({"kernel": "kv4_quantize", "shape": [131072, 1024, 128], "us": t * 1e6, "GBs": byts / t / 1e9})
    Qb, sb, zb = comet.comet_quantize_kv(KVb, 128)
    t = timed(lambda: comet.comet_dequantize_kv(Qb, sb, zb, 128))
    out.append({"kernel": "kv4_dequantize", "shape": [131072, 1024, 128], "us": t * 1e6, "GBs": byts / t / 1e9})
    del KVb, Qb, sb, zb
    # f4: static-scale activation quantize vs the dynamic one, M=K=4096, 3/32 INT8 blocks
    M, K = 4096, 4096
    bits = np.full(K // 128, 4, np.uint8)
    bits[:3] = 8
    Xa = torch.randn(M, K, device="cuda").half()
    perm = torch.randperm(K, device="cuda").int()
    sc = comet.comet_static_act_scales(comet.comet_calib_absmax(Xa), bits, perm)
    planes = comet.alloc_act_planes(M, K, bits, Xa.device)
    byts = M * K * 2 + M * (3 * 128 + 29 * 64) + (K // 128) * M * 4
    t = timed(lambda: comet.comet_quantize_act_static(Xa, bits, sc, perm, out=planes))
    out.append({"kernel": "quantize_act_static", "shape": [M, K], "us": t * 1e6, "GBs": byts / t / 1e9})
    t = timed(lambda: comet.comet_quantize_act(Xa, bits, perm, out=planes))
    out.append({"kernel": "quantize_act (dynamic)", "shape": [M, K], "us": t * 1e6, "GBs": byts / t / 1e9})
    # f3: decode attention over KV4 caches (dequant-in-attention), 32 heads x 128, T tokens, group 128
    for T in (8192, 32768):
        H = 32
        Kd = comet.comet_quantize_kv(torch.randn(T, H * 128, device="cuda").half(), 128)
        Vd = comet.comet_quantize_kv(torch.randn(T, H * 128, device="cuda").half(), 128)
        qh = torch.randn(H, 128, device="cuda").half()
        ws = torch.empty(comet.lib().comet_attention_kv4_workspace_bytes(T, H), dtype=torch.uint8, device="cuda")
        t = timed(lambda: comet.comet_attention_kv4(qh, Kd, Vd, 128, 128 ** -0.5, workspace=ws))
        byts = 2 * (T * H * 64 + (T // 128) * H * 128 * 5)
        out.append({"kernel": "attention_kv4", "shape": [T, H, 128], "us": t * 1e6, "GBs": byts / t / 1e9})
    for o in out:
        o["frac_of_hbm"] = o["GBs"] / pk
        print(json.dumps(o))


if __name__ == "__main__":
    main()
