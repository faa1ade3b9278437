set -x; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout -s KILL 400 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_7b.json 2> gpurun_out/bench_7b.err; echo rc=$?
timeout -s KILL 200 python bench.py --config llama2-7b-decode --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_7b_decode.json 2> gpurun_out/bench_7b_decode.err; echo rc=$?
timeout -s KILL 300 python bench.py --config llama3-70b --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_70b.json 2> gpurun_out/bench_70b.err; echo rc=$?
timeout -s KILL 300 python bench.py --config llama3-70b-decode --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_70b_decode.json 2> gpurun_out/bench_70b_decode.err; echo rc=$?
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k full_size > gpurun_out/parity_full.log 2>&1; echo rc=$?
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_7b.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo rc=$?
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:w4ax_gemm -s 6 -c 2 -o gpurun_out/prof_gemm_7b python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo rc=$?
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:quantize_act -s 6 -c 1 -o gpurun_out/prof_quant_7b python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_q.log 2>&1; echo rc=$?
cat gpurun_out/bench_7b.json gpurun_out/bench_7b_decode.json gpurun_out/bench_70b.json gpurun_out/bench_70b_decode.json
tail -3 gpurun_out/parity_full.log
