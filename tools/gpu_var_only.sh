mkdir -p gpurun_out; bash tools/gpu_variants2.sh
