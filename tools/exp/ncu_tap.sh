#!/bin/bash
for f in 1 0; do
LC_SUBPIX_FUSED=$f ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/tap_launch_b_$f.csv python tools/profile_step.py B 1 > gpurun_out/tap_ncu_b_$f.log 2>&1
LC_SUBPIX_FUSED=$f ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/tap_launch_d_$f.csv python tools/profile_step.py D 1 > gpurun_out/tap_ncu_d_$f.log 2>&1
done
ls -la gpurun_out/tap_*
