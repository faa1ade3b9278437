"""a7 schedule ablation (the paper's Fig 9 analogue) for the
prefill kernel: persistent CTA pairs (74, the product schedule) vs a
non-persistent grid of one CTA pair per tile ("static": the hardware hands
tiles to SM pairs in waves) vs half the SM pairs.  Per-channel weights,
~10% INT8 blocks; CUDA events, L2 flushed.  Y is identical in all three."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_12168_b200 import comet
from tools.gemm_sweep import run

L = comet.lib()
L.comet_debug_set_pf_clusters.argtypes = [ctypes.c_int]
shapes = [(4096, 11008, 4096, 3), (8192, 28672, 4096, 3), (8192, 4096, 14336, 11), (8192, 57344, 8192, 6)]
for M, N, K, n8 in shapes:
    tiles = ((M + 255) // 256) * ((N + 191) // 192)
    for name, n in (("persistent-74", 0), ("static-per-tile", tiles), ("persistent-37", 37)):
        L.comet_debug_set_pf_clusters(n)
        r = run(M, N, K, n8, group="K", reps=10)
        print(json.dumps({"schedule": name, "tiles": tiles, "waves": round(tiles / 74, 2), **r}))
L.comet_debug_set_pf_clusters(0)
