"""Prefill tile-raster ablation: token tiles per raster group (1 = weight tiles
fastest, m_tiles = token tiles fastest, 0 = the library's L2-budget rule)."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_12168_b200 import comet
from tools.gemm_sweep import run

L = comet.lib()
L.comet_debug_set_pf_group.argtypes = [ctypes.c_int]
shapes = [(8192, 4096, 14336, 11), (8192, 8192, 28672, 22), (8192, 28672, 4096, 3), (8192, 6144, 4096, 3),
          (8192, 4096, 4096, 3), (8192, 57344, 8192, 6), (16384, 8192, 28672, 22)]
for M, N, K, n8 in shapes:
    mt = (M + 255) // 256
    for g in (0, mt, 1, 4, 8, 16):
        if g > mt:
            continue
        L.comet_debug_set_pf_group(g)
        r = run(M, N, K, n8, group="K", reps=8)
        print(json.dumps({"group_m": g, **{k: r[k] for k in ("M", "N", "K")}, "us": round(r["us"], 1), "TOPS": round(r["TOPS"])}))
L.comet_debug_set_pf_group(0)
