"""How much of an event-timed single launch is launch/event latency? (tools only)"""
import numpy as np, torch
x = torch.empty(1024, device="cuda")
f = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def t(fn, pre=True, reps=20):
    ts = []
    for _ in range(reps):
        f.fill_(1)
        if pre:
            torch.cuda._sleep(1_000_000)
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))
one = lambda: x.add_(1)
two = lambda: (x.add_(1), x.add_(1))
four = lambda: [x.add_(1) for _ in range(4)]
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    one(); torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        one()
g4 = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(g4, stream=s):
        four()
torch.cuda.synchronize()
print({"1 kernel": t(one), "2 kernels": t(two), "4 kernels": t(four), "1 kernel no spin": t(one, pre=False),
       "graph(1)": t(g.replay), "graph(4)": t(g4.replay)})
