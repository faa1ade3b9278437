#!/bin/bash
# round-2 final evidence (second half): GPU tests, smoke, benches (8B default with CPU baseline, 70B, 70B decode,
# 7B, reference arm), quantizer sweeps, ncu launch list + full captures, compute-sanitizer
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; echo test_rc=$?; tail -2 gpurun_out/gputest.log
timeout -s KILL 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
timeout -s KILL 900 python bench.py > gpurun_out/bench_r2_8b.json 2> gpurun_out/bench_r2_8b.err; echo b8_rc=$?
timeout -s KILL 900 python bench.py --config llama3-70b --no-cpu-baseline > gpurun_out/bench_r2_70b.json 2> gpurun_out/bench_r2_70b.err; echo b70_rc=$?
timeout -s KILL 900 python bench.py --config llama3-70b-decode --no-cpu-baseline > gpurun_out/bench_r2_70b_decode.json 2> gpurun_out/bench_r2_70b_decode.err; echo b70d_rc=$?
timeout -s KILL 900 python bench.py --config llama2-7b --no-cpu-baseline > gpurun_out/bench_r2_7b.json 2> gpurun_out/bench_r2_7b.err; echo b7_rc=$?
timeout -s KILL 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_r2_ref.json 2> gpurun_out/bench_r2_ref.err; echo ref_rc=$?
timeout -s KILL 600 python tools/quant_sweep.py > gpurun_out/quant_sweep_r2.txt 2>&1; echo qs_rc=$?
timeout -s KILL 600 python tools/quant_sweep.py '[[8192, 4096, 3], [8192, 14336, 11], [16384, 8192, 6], [8192, 28672, 22]]' fmpq >> gpurun_out/quant_sweep_r2.txt 2>&1; echo qsf_rc=$?
timeout -s KILL 600 python tools/aux_bench.py > gpurun_out/aux_bench_r2.txt 2>&1; echo aux_rc=$?
timeout -s KILL 900 python tools/m_sweep.py > gpurun_out/m_sweep_r2b.txt 2>&1; echo msw_rc=$?
bash tools/profile_round.sh
