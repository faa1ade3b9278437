#!/bin/bash
# round-end evidence: the whole GPU test suite, the benches, the ncu profiles
mkdir -p gpurun_out
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/smoke.log
timeout -s KILL 1200 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo gpu_tests_rc=$?; tail -3 gpurun_out/gpu_tests.log
timeout -s KILL 400 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo default rc=$?; tail -c 1500 gpurun_out/bench_default.json
mkdir -p gpurun_out
run() {  # name, args...
  name=$1; shift
  timeout -s KILL 400 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; echo "$name rc=$?"
  python - "$name" << 'PY'
import json,sys
try:
    d=json.load(open(f"gpurun_out/bench_{sys.argv[1]}.json"))
    r=d["roofline"]
    print(f"  {d['value']:.1f} TOPS  {d['ms_per_step']:.3f} ms  gemm_us={[round(x,1) for x in d['gemm_us']]}  roof={r['bound']} {r['achieved']:.0f}/{r['peak']:.0f} {r['unit']} frac={r['frac']:.3f}  e2e={d['e2e']['value']:.1f}  clocks={d['clocks']}")
except Exception as e:
    print("  parse error", e)
PY
}
run 7b --steps 20 --warmup 5
run 7b_g128 --group 128 --steps 20 --warmup 5 --no-cpu-baseline
run 7b_decode --config llama2-7b-decode --steps 50 --warmup 5 --no-cpu-baseline
run 70b --config llama3-70b --steps 10 --warmup 3 --no-cpu-baseline
run 70b_decode --config llama3-70b-decode --steps 20 --warmup 3 --no-cpu-baseline
if [ "$1" == "ncu" ]; then
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:w4ax_gemm -s 6 -c 2 -o gpurun_out/prof_gemm python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu rc=$?
fi

bash tools/profile_round.sh
run 7b_xw --steps 20 --warmup 5 --no-cpu-baseline --expanded-weights
run 70b_xw --config llama3-70b --steps 10 --warmup 3 --no-cpu-baseline --expanded-weights
