"""Whole-step device time without per-kernel events (so PDL overlap between
the quantizer and the GEMM is not broken by event records) -- tools only."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2410_12168_b200 import comet, synth

def main(cfg_name, reps=20):
    cfg = bench.CONFIGS[cfg_name]
    dev = torch.device("cuda")
    M = cfg["M"]
    L = []
    for li, ((N, K), n8) in enumerate(zip(cfg["layers"], cfg["n8"])):
        p = synth.make_problem(M, N, K, n8=n8, seed=100 + li)
        perm = torch.from_numpy(p["perm"]).to(dev)
        bits = comet.BlockBits(p["bits"])
        Wq, Sw = comet.comet_pack_weight(torch.from_numpy(p["W"]).to(dev), perm, K)
        X = torch.from_numpy(p["X"]).to(dev)
        L.append(dict(X=X, perm=perm, bits=bits, Wq=Wq, Sw=Sw, K=K, planes=comet.alloc_act_planes(M, K, bits, dev),
                      Y=torch.empty((M, N), dtype=torch.float16, device=dev),
                      ws=comet.new_workspace(comet.comet_w4ax_gemm_workspace_bytes(M, N, K), dev)))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    def step():
        for l in L:
            q = comet.comet_quantize_act(l["X"], l["bits"], l["perm"], out=l["planes"])
            comet.comet_w4ax_gemm(*q, l["bits"], l["Wq"], l["Sw"], l["K"], out=l["Y"], workspace=l["ws"])
    ts = []
    for i in range(reps + 3):
        flush.fill_(1)
        torch.cuda._sleep(2_000_000)
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); step(); b.record()
        torch.cuda.synchronize()
        if i >= 3: ts.append(a.elapsed_time(b) * 1e3)
    print(json.dumps({"config": cfg_name, "step_us_median": float(np.median(ts)), "min": float(np.min(ts))}))

if __name__ == "__main__":
    for c in sys.argv[1:] or ["llama2-7b", "llama3-70b-decode", "llama2-7b-decode"]:
        main(c)
