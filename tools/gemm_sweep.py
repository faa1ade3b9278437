"""Time comet_w4ax_gemm alone over shapes (CUDA events, L2 flushed between reps)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2410_12168_b200 import comet, synth

def run(M, N, K, n8, group, reps=20, flush_mode="write"):
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
    tiny = torch.zeros(1024, device=dev)
    ts = []
    for i in range(reps + 3):
        if flush_mode == "write":
            flush.fill_(1)
        else:  # read-only sweep: L2 ends full of clean lines (no write-back debt)
            torch.sum(flush.view(torch.int64), dtype=torch.int64)
        torch.cuda._sleep(1_000_000)  # host enqueues ahead: time the kernel, not the launch path
        tiny.add_(1)  # the ~5 us event->first-launch floor lands before `a` (tools/event_overhead.py)
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
    mode = sys.argv[2] if len(sys.argv) > 2 else "write"
    for s in shapes:
        print(json.dumps(dict(run(*s, group="K", flush_mode=mode), flush=mode)))


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


def roles(M, N, K, n8, cta=0):
    import ctypes
    L = comet.lib()
    L.comet_debug_cta_times.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
    L.comet_debug_role_cycles.argtypes = [ctypes.c_void_p]
    L.comet_debug_cta_times(cta + 1, None, 0)
    run(M, N, K, n8, "K", reps=1)
    L.comet_debug_cta_times(0, None, 0)
    buf = (ctypes.c_ulonglong * 16)()
    L.comet_debug_role_cycles(buf)
    a = np.array(buf[:], dtype=np.int64).reshape(4, 4)
    names = [("producer", "wait empty", "wait sempty"), ("mma", "wait tempty", "wait expd"),
             ("expand g0", "wait full", "wait aempty"), ("epilogue", "wait sfull", "wait tfull")]
    print(f"M={M} N={N} K={K} CTA{cta} roles (cycles):")
    for (n, w0, w1), row in zip(names, a):
        print(f"  {n:10s} total {row[2]:8d}  {w0} {row[0]:8d} ({row[0]/max(row[2],1):.0%})  {w1} {row[1]:8d} ({row[1]/max(row[2],1):.0%})"
              + (f"  fixup {row[3]:8d}" if row[3] else ""))


def slowest_roles(M, N, K, n8):
    import ctypes
    L = comet.lib()
    L.comet_debug_cta_times.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
    L.comet_debug_cta_times(1, None, 0)
    run(M, N, K, n8, "K", reps=1)
    buf = (ctypes.c_ulonglong * (3 * 1024))()
    L.comet_debug_cta_times(0, buf, 148)
    a = np.array(buf[: 3 * 148], dtype=np.int64).reshape(148, 3)
    d = (a[:, 1] - a[:, 0]) / 1e3
    o = np.argsort(-d)
    print("durations us (slowest 8):", [(int(i), round(float(d[i]), 1)) for i in o[:8]], "median", round(float(np.median(d)), 1))
    for c in list(o[:2]) + [int(np.argsort(d)[74])]:
        roles(M, N, K, n8, int(c))


def launch_gap(M, N, K, n8, reps=20):
    """events around `reps` back-to-back launches (no flush) vs one launch; plus CTA start spread"""
    dev = torch.device("cuda")
    bits = comet.BlockBits(synth.block_bits_for(K, n8))
    W = torch.randn(N, K, device=dev).half() / K ** 0.5
    X = torch.randn(M, K, device=dev).half()
    Wq, Sw = comet.comet_pack_weight(W, None, K)
    planes = comet.comet_quantize_act(X, bits)
    ws = comet.new_workspace(comet.comet_w4ax_gemm_workspace_bytes(M, N, K), dev)
    Y = torch.empty(M, N, dtype=torch.float16, device=dev)
    f = lambda: comet.comet_w4ax_gemm(*planes, bits, Wq, Sw, K, out=Y, workspace=ws)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    torch.cuda._sleep(2_000_000)
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(reps):
        f()
    b.record()
    torch.cuda.synchronize()
    per = a.elapsed_time(b) * 1e3 / reps
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        f()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                f()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    pg = a.elapsed_time(b) * 1e3 / reps
    ok = True
    print(json.dumps({"M": M, "N": N, "K": K, "us_per_launch_b2b": per, "us_per_launch_graph": pg}))


def trace(M, N, K, n8, cta=0, units=24):
    """per-unit event timeline (cycles from the first W issue) of one CTA"""
    import ctypes
    L = comet.lib()
    L.comet_debug_cta_times.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
    L.comet_debug_trace.argtypes = [ctypes.c_void_p]
    buf = (ctypes.c_ulonglong * 2048)()
    L.comet_debug_trace(buf)  # clear-less: events of untraced units stay stale, print only < units
    L.comet_debug_cta_times(cta + 1, None, 0)
    run(M, N, K, n8, "K", reps=1)
    L.comet_debug_cta_times(0, None, 0)
    L.comet_debug_trace(buf)
    a = np.array(buf[:], dtype=np.int64).reshape(32, 64)
    t0 = a[0, 0]
    names = ["Wiss", "Xiss", "arrive", "expd", "mma", "accrdy", "accrel", "retire", "epitop", "sxrdy"]
    print(f"M={M} N={N} K={K} CTA{cta} trace (cycles rel. first W issue):")
    print("unit " + " ".join(f"{n:>7s}" for n in names))
    for i in range(units):
        print(f"{i:4d} " + " ".join(f"{a[e, i] - t0:7d}" for e in range(10)))


def trace3(M, N, K, n8, cta=0, steps=40):
    """TMEM-A prefill kernel (gemm_pf.cuh): per-step event timeline of one CTA"""
    import ctypes
    L = comet.lib()
    L.comet_debug_cta_times.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
    L.comet_debug_trace.argtypes = [ctypes.c_void_p]
    buf = (ctypes.c_ulonglong * 2048)()
    L.comet_debug_cta_times(cta + 1, None, 0)
    run(M, N, K, n8, "K", reps=1)
    L.comet_debug_cta_times(0, None, 0)
    L.comet_debug_trace(buf)
    a = np.array(buf[:], dtype=np.int64).reshape(32, 64)
    t0 = a[0, 0]
    names = ["Ptop", "staged", "tfull0", "prom0", "-", "-", "mrdy", "mma0", "temty", "Wiss", "Xiss", "sxrdy"]
    print(f"M={M} N={N} K={K} CTA{cta} pf trace (cycles rel. first P iteration; staged = block g+2 staged):")
    print("step " + " ".join(f"{n:>7s}" for n in names))
    for i in range(steps):
        print(f"{i:4d} " + " ".join(f"{a[e, i] - t0:7d}" for e in range(12)))
    print("MMA issue sub-events (temty, after 1st MMA, after 4th MMA, after commits), steps 8-15:")
    for i in range(8, 16):
        print(f"  {i:3d} {a[8, i] - t0:7d} {a[4, 32 + i] - t0:7d} {a[5, 32 + i] - t0:7d} {a[7, i] - t0:7d}")
    print("block: W-prod issue, X-prod issue, staging lfull seen, staging start (mdone seen), LDS landed, tokens zext done, [EV2: STTM issued, weights done], staged")
    for i in range(8, 16):
        print(f"  {i:3d} {a[14, i] - t0:7d} {a[15, i] - t0:7d} {a[12, i] - t0:7d} {a[10, i] - t0:7d} {a[16, i] - t0:7d} {a[13, i] - t0:7d} [{a[6, i] - t0:7d} {a[9, i] - t0:7d}] {a[1, i] - t0:7d}")
    for e, st in ((4, 10), (5, 11)):
        print(f"step {st} per-warp release (CTA pair, leader then partner):")
        print("  " + " ".join(f"{a[e, w] - t0:6d}" for w in range(12)))
        print("  " + " ".join(f"{a[e, 16 + w] - t0:6d}" for w in range(12)))


def trace2(M, N, K, n8, cta=0, steps=40):
    """prefill (CTA-pair) kernel: per-step event timeline of one CTA's compute warp 0"""
    import ctypes
    L = comet.lib()
    L.comet_debug_cta_times.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
    L.comet_debug_trace.argtypes = [ctypes.c_void_p]
    buf = (ctypes.c_ulonglong * 2048)()
    L.comet_debug_cta_times(cta + 1, None, 0)
    run(M, N, K, n8, "K", reps=1)
    L.comet_debug_cta_times(0, None, 0)
    L.comet_debug_trace(buf)
    a = np.array(buf[:], dtype=np.int64).reshape(32, 64)
    t0 = a[0, 0]
    names = ["iter", "fullnx", "expdnx", "sxrdy", "accrdy", "promdn", "mma", "prod"]
    print(f"M={M} N={N} K={K} CTA{cta} prefill trace (cycles rel. first iteration; fullnx/expdnx = step g):")
    print("step " + " ".join(f"{n:>7s}" for n in names))
    for i in range(steps):
        print(f"{i:4d} " + " ".join(f"{a[e, i] - t0:7d}" for e in range(8)))


def trace_pf(M, N, K, n8, cta=0, steps=64, group="K"):
    """fp8-promotion prefill kernel (gemm_pf.cuh): per-block event timeline of one (leader) CTA"""
    import ctypes
    L = comet.lib()
    L.comet_debug_cta_times.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
    L.comet_debug_trace.argtypes = [ctypes.c_void_p]
    buf = (ctypes.c_ulonglong * 2048)()
    L.comet_debug_cta_times(cta + 1, None, 0)
    run(M, N, K, n8, group, reps=1)
    L.comet_debug_cta_times(0, None, 0)
    L.comet_debug_trace(buf)
    a = np.array(buf[:], dtype=np.int64).reshape(32, 64)
    t0 = a[4, 0]
    names = ["Ptop", "Ptfull", "Prel", "Pend", "Mtop", "Mrdy", "Mtemp", "Mcomm", "Stop", "Slfull", "Smdone",
             "Srdy", "Wiss", "Xiss", "P19tf", "P19rel"]
    print(f"M={M} N={N} K={K} g={group} CTA{cta} pf trace (cycles rel. first MMA-warp iteration):")
    print("step " + " ".join(f"{n:>7s}" for n in names))
    for i in range(steps):
        print(f"{i:4d} " + " ".join(f"{a[e, i] - t0:7d}" for e in range(16)))
    d = np.diff(a[7, 8:steps])
    print(f"MMA commit interval steps 8..{steps - 1}: median {np.median(d):.0f} mean {d.mean():.0f} cycles")
    print("MMA issue detail: temty, elected, after MMA0, after MMA3, after commit0, after commit1; then P19 tfull/release")
    for i in range(8, 24):
        print(f"  {i:3d} " + " ".join(f"{a[e, i] - t0:7d}" for e in (6, 16, 17, 18, 19, 7, 15)))
    print("accumulator hand-off, steps 16..19, CTA0's 12 promotion warps: seen / released (rel. the step's commit)")
    for i in range(16, 20):
        r = a[25 + i - 16]
        seen = [int(r[2 * w] - a[7, i]) for w in range(12)]
        rel = [int(r[2 * w + 1] - a[7, i]) for w in range(12)]
        print(f"  {i:3d} commit {a[7, i] - t0:7d}  MMA sees free (step+2) +{a[6, i + 2] - a[7, i]}")
        print("       seen " + " ".join(f"{x:5d}" for x in seen))
        print("       rel  " + " ".join(f"{x:5d}" for x in rel))
    print("staging detail: mdone seen, LDS landed, weights stored, tokens st issued, proxy fence done, st wait done, ready arrived")
    for i in range(8, 24):
        print(f"  {i:3d} " + " ".join(f"{a[e, i] - t0:7d}" for e in (10, 20, 21, 22, 23, 24, 11)))
