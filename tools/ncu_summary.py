"""Summarise ncu captures into profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py ROUND

Reads gpurun_out/launches.csv and gpurun_out/prof_*_full.ncu-rep, writes
profiles/ncu_launches_<ROUND>.csv (the launch list of the bench command),
profiles/ncu_summary_<ROUND>.md (key counters per captured kernel) and
profiles/ncu_traffic.json (dram bytes per GEMM launch, read by bench.py).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    ("gpu__time_duration.sum", "duration (us)", 1e-3),  # base unit ns
    ("sm__cycles_active.avg", "SM active cycles (avg)", 1),
    ("dram__bytes_read.sum", "DRAM read (MB)", 1e-6),   # base unit bytes
    ("dram__bytes_write.sum", "DRAM write (MB)", 1e-6),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active (%)", 1),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe active (%)", 1),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active (%)", 1),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy (%)", 1),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts (% of peak)", 1),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts", 1),
    ("launch__registers_per_thread", "registers/thread", 1),
    ("launch__grid_size", "grid", 1),
    ("launch__block_size", "block", 1),
]


UNIT = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "ns": 1.0, "us": 1e3, "ms": 1e6, "s": 1e9,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def raw(rep):
    """per-kernel dict of counters in base units (ns, bytes)"""
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        d = {}
        for h, u, v in zip(hdr, units, r):
            x = num(v)
            d[h] = x * UNIT[u] if (x is not None and u in UNIT) else (x if x is not None else v)
        out.append(d)
    return out


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def main(rnd):
    os.makedirs(PROF, exist_ok=True)
    md = [f"# ncu summary, round {rnd}", "",
          "Captured under gpurun on one B200 with `ncu --set full --clock-control none` "
          "(cold caches, serialised replays: durations are longer than the bench's "
          "CUDA-event numbers; compare shares and counters, not absolutes).", ""]
    traffic = {}
    for tag, rep in [("prefill GEMM (LLaMA-3-8B gate_up 28672x4096 and down 4096x14336, M=8192, per-channel weight scales)", "prof_gemm_full"),
                     ("quantize_act: quantize_lane_kernel (LLaMA-3-8B, M=8192, FMPQ permutation; layers 2 and 3)", "prof_quant_full"),
                     ("decode GEMM (LLaMA-3-70B, M=16; layers 2 and 3)", "prof_decode_full")]:
        path = os.path.join(OUT, rep + ".ncu-rep")
        if not os.path.exists(path):
            continue
        kernels = raw(path)
        md.append(f"## {tag}  (`{rep}.ncu-rep`)")
        md.append("")
        md.append("| counter | " + " | ".join(f"launch {i}" for i in range(len(kernels))) + " |")
        md.append("|---|" + "---|" * len(kernels))
        md.append("| kernel | " + " | ".join(str(k.get("Kernel Name", "?"))[:48] for k in kernels) + " |")
        for key, name, scale in KEYS:
            vals = []
            for k in kernels:
                v = k.get(key)
                vals.append("-" if not isinstance(v, float) else (f"{v * scale:.4g}"))
            md.append(f"| {name} | " + " | ".join(vals) + " |")
        md.append("")
        if rep == "prof_gemm_full":
            for i, k in enumerate(kernels):
                rd, wr = k.get("dram__bytes_read.sum"), k.get("dram__bytes_write.sum")
                if isinstance(rd, float) and isinstance(wr, float):
                    traffic[f"layer{i + 2}"] = rd + wr  # launches 0, 1 = layers 2 (gate_up), 3 (down)
    with open(os.path.join(PROF, f"ncu_summary_{rnd}.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    if traffic:
        with open(os.path.join(PROF, "ncu_traffic.json"), "w") as f:
            json.dump({"llama3-8b/gchannel": traffic, "_note": "dram__bytes_read.sum + dram__bytes_write.sum per GEMM launch "
                       "(bytes), from one ncu --set full capture (" + rnd + ")"}, f, indent=1)
    # launch list
    src = os.path.join(OUT, "launches.csv")
    if os.path.exists(src):
        rows = list(csv.reader(open(src)))
        start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
        hdr = rows[start]
        ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
        lines = [("id", "kernel", "time_ns")]
        tot = {}
        for r in rows[start + 1:]:
            if len(r) == len(hdr):
                name = r[ki].split("(")[0].split("<")[0].replace("void ", "").strip()
                t = num(r[vi])
                lines.append((r[0], name, r[vi]))
                tot[name] = tot.get(name, 0) + (t or 0)
        with open(os.path.join(PROF, f"ncu_launches_{rnd}.csv"), "w") as f:
            csv.writer(f).writerows(lines)
        s = sum(tot.values())
        with open(os.path.join(PROF, f"ncu_summary_{rnd}.md"), "a") as f:
            f.write("## launch list of `bench.py --steps 2 --warmup 3` (all kernels, ncu gpu__time_duration)\n\n")
            f.write("| kernel | total us | share |\n|---|---|---|\n")
            for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
                f.write(f"| {k} | {v / 1e3:.1f} | {v / s:.1%} |\n")
    print(open(os.path.join(PROF, f"ncu_summary_{rnd}.md")).read())


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r1")
