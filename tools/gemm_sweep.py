"""Time comet_w4ax_gemm alone over shapes (CUDA events, L2 flushed between reps)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2410_12168_b200 import comet, synth

def run(M, N, K, n8, group, reps=20):
    dev = torch.device("cuda")
    rng = np.random.default_rng(0)
    bits = comet.BlockBits(synth.block_bits_for(K, n8))
    W = torch.randn(N, K, device=dev).half() / K ** 0.5
    X = torch.randn(M, K, device=dev).half()
    g = K if group == "K" else 128
    Wq, Sw = comet.comet_pack_weight(W, None, g)
    planes = comet.comet_quantize_act(X, bits)
    ws = comet.new_workspace(comet.comet_w4ax_gemm_workspace_bytes(M, N, K), dev)
    Y = torch.empty(M, N, dtype=torch.float16, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ts = []
    for i in range(reps + 3):
        flush.fill_(1)
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); comet.comet_w4ax_gemm(*planes, bits, Wq, Sw, g, out=Y, workspace=ws); b.record()
        torch.cuda.synchronize()
        if i >= 3: ts.append(a.elapsed_time(b))
    t = float(np.median(ts)) * 1e-3
    nb = K // 128
    byts = N * K / 2 + 4 * N * (K // g) + M * (128 * n8 + 64 * (nb - n8)) + 4 * M * nb + 2 * M * N
    return {"M": M, "N": N, "K": K, "us": t * 1e6, "TOPS": 2 * M * N * K / t / 1e12, "GBs": byts / t / 1e9}

if __name__ == "__main__":
    shapes = json.loads(sys.argv[1]) if len(sys.argv) > 1 else [[16, 4096, 4096, 3], [16, 11008, 4096, 3], [16, 57344, 8192, 6], [16, 8192, 28672, 22], [1, 4096, 4096, 3], [64, 4096, 4096, 3], [128, 11008, 4096, 3]]
    for s in shapes:
        print(json.dumps(run(*s, group="K")))


def cta_times(M, N, K, n8):
    import ctypes
    L = comet.lib()
    L.comet_debug_cta_times.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
    L.comet_debug_cta_times(1, None, 0)
    run(M, N, K, n8, "K", reps=1)
    buf = (ctypes.c_ulonglong * (3 * 1024))()
    L.comet_debug_cta_times(0, buf, 148)
    a = np.array(buf[: 3 * 148], dtype=np.int64).reshape(148, 3)
    t0 = a[:, 0].min()
    st, en = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3
    print(f"M={M} N={N} K={K}: start us min/med/max {st.min():.1f}/{np.median(st):.1f}/{st.max():.1f}; "
          f"dur us min/med/max {(en-st).min():.1f}/{np.median(en-st):.1f}/{(en-st).max():.1f}; end max {en.max():.1f}; "
          f"distinct sms {len(set(a[:,2]))}")
    order = np.argsort(st)
    print("  latest starts:", [(int(i), round(float(st[i]),1), int(a[i,2])) for i in order[-6:]])


def slow_ctas(M, N, K, n8):
    import ctypes
    L = comet.lib()
    L.comet_debug_cta_times.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
    for rep in range(3):
        L.comet_debug_cta_times(1, None, 0)
        run(M, N, K, n8, "K", reps=1)
        buf = (ctypes.c_ulonglong * (3 * 1024))()
        L.comet_debug_cta_times(0, buf, 148)
        a = np.array(buf[: 3 * 148], dtype=np.int64).reshape(148, 3)
        d = (a[:, 1] - a[:, 0]) / 1e3
        o = np.argsort(-d)
        print(f"M={M} N={N}: slowest", [(int(i), round(float(d[i]), 1), int(a[i, 2])) for i in o[:5]], "median", round(float(np.median(d)), 1))


def roles(M, N, K, n8):
    import ctypes
    L = comet.lib()
    L.comet_debug_cta_times.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
    L.comet_debug_role_cycles.argtypes = [ctypes.c_void_p]
    L.comet_debug_cta_times(1, None, 0)
    run(M, N, K, n8, "K", reps=1)
    L.comet_debug_cta_times(0, None, 0)
    buf = (ctypes.c_ulonglong * 12)()
    L.comet_debug_role_cycles(buf)
    a = np.array(buf[:], dtype=np.int64).reshape(4, 3)
    names = [("producer", "wait empty", "wait sempty"), ("mma", "wait tempty", "wait expd"),
             ("expand g0", "wait full", "wait aempty"), ("epilogue", "wait sfull", "wait tfull")]
    print(f"M={M} N={N} K={K} CTA0 roles (cycles):")
    for (n, w0, w1), row in zip(names, a):
        print(f"  {n:10s} total {row[2]:8d}  {w0} {row[0]:8d} ({row[0]/max(row[2],1):.0%})  {w1} {row[1]:8d} ({row[1]/max(row[2],1):.0%})")
