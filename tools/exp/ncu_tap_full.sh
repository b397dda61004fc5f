#!/bin/bash
ncu --set full --clock-control none --import-source on -k regex:tap_tc --launch-skip 0 --launch-count 1 \
    -o gpurun_out/tap_head python tools/profile_step.py B 1 > gpurun_out/tap_full_head.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tap_tc --launch-skip 4 --launch-count 1 \
    -o gpurun_out/tap_dec python tools/profile_step.py B 1 > gpurun_out/tap_full_dec.log 2>&1
ls -la gpurun_out/tap_head* gpurun_out/tap_dec*
