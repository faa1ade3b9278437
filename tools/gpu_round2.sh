#!/bin/bash
# round-2 evidence: GPU tests, default bench (+ 70B configs), ncu captures
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; echo test_rc=$?; tail -2 gpurun_out/gputest.log
timeout -s KILL 900 python bench.py > gpurun_out/bench_r2_8b.json 2> gpurun_out/bench_r2_8b.err; echo b8_rc=$?
timeout -s KILL 900 python bench.py --config llama3-70b --no-cpu-baseline > gpurun_out/bench_r2_70b.json 2> gpurun_out/bench_r2_70b.err; echo b70_rc=$?
timeout -s KILL 900 python bench.py --config llama3-70b-decode --no-cpu-baseline > gpurun_out/bench_r2_70b_decode.json 2> gpurun_out/bench_r2_70b_decode.err; echo b70d_rc=$?
timeout -s KILL 900 python bench.py --config llama2-7b --no-cpu-baseline > gpurun_out/bench_r2_7b.json 2> gpurun_out/bench_r2_7b.err; echo b7_rc=$?
timeout -s KILL 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_r2_ref.json 2> gpurun_out/bench_r2_ref.err; echo ref_rc=$?
bash tools/profile_round.sh
