"""Summarise an ncu report: top stall reasons, samples per SASS opcode -- tools only.
    python tools/ncu_stalls.py report.ncu-rep"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)))
h, v = raw[0], raw[2]
st = []
for i, k in enumerate(h):
    if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
        try: st.append((float(v[i].replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError: pass
tot = sum(x for x, _ in st) or 1
print("stall reasons (share of samples):")
for x, k in sorted(st, reverse=True)[:10]: print(f"  {k:28s} {100 * x / tot:5.1f}%")
src = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout)))
hh = src[1] if len(src) > 1 and "Source" in src[1] else src[0]
rows = src[2:] if hh is src[1] else src[1:]
si, ni, ei = hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)"), hh.index("Instructions Executed")
by = collections.Counter(); ex = collections.Counter()
for r in rows:
    if len(r) <= max(si, ni, ei): continue
    op = r[si].strip().split()
    if not op: continue
    o = op[0] if not op[0].startswith("@") else op[1]
    try: by[o] += float(r[ni] or 0); ex[o] += float(r[ei] or 0)
    except ValueError: pass
t = sum(by.values()) or 1
te = sum(ex.values()) or 1
print("samples / executed warp-instructions per opcode:")
for o, x in by.most_common(25): print(f"  {o:24s} {100 * x / t:5.1f}%  exec {100 * ex[o] / te:5.1f}%")
