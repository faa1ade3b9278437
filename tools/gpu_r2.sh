set -x; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout -s KILL 120 ./tools/microbench > gpurun_out/microbench.txt 2>&1; echo mb rc=$?
bash tools/gpu_bench.sh
