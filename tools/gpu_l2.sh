mkdir -p gpurun_out; timeout -s KILL 120 ./tools/mb_l2 > gpurun_out/mb_l2.txt 2>&1; timeout -s KILL 120 ./tools/mb_l2mc > gpurun_out/mb_l2mc.txt 2>&1; cat gpurun_out/mb_l2.txt gpurun_out/mb_l2mc.txt
