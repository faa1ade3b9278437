"""One comet_quantize_act call per (shape, permutation kind) for ncu -- tools only.
    python tools/prof_quant.py M K n8 kind[fmpq|random|none] [reps]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2410_12168_b200 import comet, synth

M, K, n8, kind = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 1
p = synth.make_problem(8, 128, K, n8=n8, seed=1)
perm = None if kind == "none" else (p["perm"] if kind == "fmpq" else np.random.default_rng(0).permutation(K).astype(np.int32))
dev = torch.device("cuda")
X = torch.randn(M, K, device=dev).half()
bits = comet.BlockBits(p["bits"])
pt = None if perm is None else torch.from_numpy(perm).to(dev)
for _ in range(reps):
    comet.comet_quantize_act(X, bits, pt)
torch.cuda.synchronize()
