#!/bin/bash
# Only the `ncu --set full` captures of tools/refresh_profiles_r02.sh.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for spec in "stem 0" "d0 1"; do set -- $spec
  ncu --set full --clock-control none --import-source on -k regex:conv_tc --launch-skip $2 --launch-count 1 \
      -o gpurun_out/full_c_$1 -f python tools/profile_step.py C 1 > gpurun_out/ncu_full_c_$1.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:tap_tc --launch-skip 0 --launch-count 1 \
    -o gpurun_out/full_c_head -f python tools/profile_step.py C 1 > gpurun_out/ncu_full_c_head.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tap_tc --launch-skip 25 --launch-count 1 \
    -o gpurun_out/full_c_dec -f python tools/profile_step.py C 1 > gpurun_out/ncu_full_c_dec.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv_tc --launch-skip 2 --launch-count 1 \
    -o gpurun_out/full_d_dec2 -f python tools/profile_step.py D 1 > gpurun_out/ncu_full_d_dec2.log 2>&1
# u0 of step 0 (the largest conv): the last conv launch of run 1's step 0 before the head
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:conv_tc --csv \
    --log-file gpurun_out/conv_list_c.csv python tools/profile_step.py C 1 > /dev/null 2>&1
ls -la gpurun_out/full_*.ncu-rep
