mkdir -p gpurun_out; bash tools/profile_round.sh; timeout -s KILL 900 python bench.py > gpurun_out/bench_r2_8b_ch.json 2> gpurun_out/bench_r2_8b_ch.err; echo b8_rc=$?
