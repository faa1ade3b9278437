"""M sweep of the W4Ax GEMM (decode kernel for M <= 128, CTA-pair prefill
above) on LLaMA-3-70B gate_up (57344 x 8192) and LLaMA-3-8B gate_up
(28672 x 4096), per-channel and group-128 weight scales: time, TOPS, GB/s
and the fractions of the measured HBM and INT8 peaks (MEASURED_PEAKS.json)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.gemm_sweep import run

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
hbm, i8 = pk["hbm_gbs"], 2 * pk["bf16_tflops"]
for N, K, n8 in ((57344, 8192, 6), (28672, 4096, 3)):
    for group in ("K", "128"):
        for M in (1, 16, 32, 64, 128, 129, 256, 512, 1024, 2048, 4096, 8192):
            r = run(M, N, K, n8, group=group, reps=10)
            print(json.dumps({**r, "group": group, "frac_hbm": round(r["GBs"] / hbm, 3),
                              "frac_int8": round(r["TOPS"] / i8, 3)}))
