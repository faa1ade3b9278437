"""INT8-block fraction sweep (0..50%) x decode/prefill M on the
LLaMA-3-70B MLP shapes, GEMM-only (tools/gemm_sweep.run: CUDA events, L2
flushed, median of 20).  The slope of time vs the number of INT8 blocks gives
the measured cost of an INT8 block relative to an INT4 block on B200
(a7: "split so every SM gets equal *measured* cost")."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np  # noqa: E402
import gemm_sweep  # noqa: E402

FRACS = [0.0, 0.1, 0.2, 0.3, 0.4, 0.5]
SHAPES = [("gate_up", 57344, 8192), ("down", 8192, 28672)]
if __name__ == "__main__":
    Ms = [int(m) for m in sys.argv[1].split(",")] if len(sys.argv) > 1 else [16, 8192]
    group = sys.argv[2] if len(sys.argv) > 2 else "K"
    rows = []
    for name, N, K in SHAPES:
        nb = K // 128
        for M in Ms:
            pts = []
            for f in FRACS:
                n8 = int(round(f * nb))
                r = gemm_sweep.run(M, N, K, n8, group)
                r.update(layer=name, frac=f, n8=n8)
                print(json.dumps(r), flush=True)
                pts.append((n8, r["us"]))
                rows.append(r)
            x = np.array([p[0] for p in pts], float)
            y = np.array([p[1] for p in pts], float)
            slope, icpt = np.polyfit(x, y, 1)
            per_block4 = icpt / nb  # time per block at 0% INT8
            print(json.dumps({"layer": name, "M": M, "group": group, "us_at_0": icpt, "us_per_int8_block_extra": slope,
                              "int8_block_cost_vs_int4": (per_block4 + slope) / per_block4}), flush=True)
