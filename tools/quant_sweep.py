"""Time comet_quantize_act alone (CUDA events, L2 flushed) -- tools only."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2410_12168_b200 import comet, synth

def run(M, K, n8, perm=True, reps=20, kind="random"):
    """kind: "random" = a uniformly random permutation, "fmpq" = synth's FMPQ
    layout (planted outliers first, the rest in order)"""
    dev = torch.device("cuda")
    bits = comet.BlockBits(synth.block_bits_for(K, n8))
    X = torch.randn(M, K, device=dev).half()
    if kind == "fmpq":
        pn = synth.make_problem(8, 128, K, n8=n8, seed=1)["perm"]
    else:
        pn = np.random.default_rng(0).permutation(K).astype(np.int32)
    p = torch.from_numpy(pn).to(dev) if perm else None
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ts = []
    for i in range(reps + 3):
        flush.fill_(1)
        torch.cuda._sleep(1_000_000)
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); comet.comet_quantize_act(X, bits, p); b.record()
        torch.cuda.synchronize()
        if i >= 3: ts.append(a.elapsed_time(b))
    t = float(np.median(ts)) * 1e-3
    nb = K // 128
    byts = 2 * M * K + M * (128 * n8 + 64 * (nb - n8)) + 4 * M * nb
    return {"M": M, "K": K, "perm": kind if perm else False, "us": t * 1e6, "GBs": byts / t / 1e9}

if __name__ == "__main__":
    shapes = json.loads(sys.argv[1]) if len(sys.argv) > 1 else [[4096, 4096, 3], [8192, 8192, 6], [16384, 8192, 6], [8192, 28672, 22], [16, 8192, 6]]
    kind = sys.argv[2] if len(sys.argv) > 2 else "random"
    for s in shapes:
        for perm in (True, False):
            print(json.dumps(run(*s, perm=perm, kind=kind)))
