#!/bin/bash
# Launch list + full ncu captures of the top kernels on the c4 bench command (run under gpurun).
set -u
A="bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline"
python $A > gpurun_out/plain_c4.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python $A > gpurun_out/ncu_launch_c4.log 2>&1; echo ncu_launch=$?
ncu --set full --clock-control none --import-source on -k regex:far_const_kernel -s 200 -c 1 -o gpurun_out/farconst_c4 python $A > gpurun_out/ncu_farconst.log 2>&1; echo ncu_far=$?
ncu --set full --clock-control none --import-source on -k regex:near_stream_kernel -c 1 -o gpurun_out/near_c4 python $A > gpurun_out/ncu_near.log 2>&1; echo ncu_near=$?
ncu --set full --clock-control none --import-source on -k regex:upsample_dmma_kernel -c 1 -o gpurun_out/upsample_c4 python $A > gpurun_out/ncu_up.log 2>&1; echo ncu_up=$?
