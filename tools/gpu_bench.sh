#!/bin/bash
# parity + benches (+ optional ncu of the GEMM when $1 == ncu)
mkdir -p gpurun_out
bash tools/gpu_test.sh
for cfg in llama2-7b llama2-7b-decode llama3-70b llama3-70b-decode; do
  extra="--no-cpu-baseline"; [ "$cfg" == "llama2-7b" ] && extra=""
  timeout -s KILL 400 python bench.py --config $cfg --steps 20 --warmup 5 $extra > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err; echo "$cfg rc=$?"
  python - "$cfg" << 'PY'
import json,sys
try:
    d=json.load(open(f"gpurun_out/bench_{sys.argv[1]}.json"))
    r=d["roofline"]
    print(f"  {d['value']:.1f} TOPS  {d['ms_per_step']:.3f} ms  gemm_us={[round(x,1) for x in d['gemm_us']]}  roof={r['bound']} {r['achieved']:.0f}/{r['peak']:.0f} {r['unit']} frac={r['frac']:.3f}  clocks={d['clocks']}")
except Exception as e:
    print("  parse error", e)
PY
done
if [ "$1" == "ncu" ]; then
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:w4ax_gemm -s 6 -c 2 -o gpurun_out/prof_gemm python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu rc=$?
fi
