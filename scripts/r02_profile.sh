#!/bin/bash
# r02 evidence on one B200: baseline stage times (C2, C3), ncu --set full of the hot
# kernels at 2^23, launch list of a C2 step. Outputs under gpurun_out/r02/$1.
T=${1:-p}; D=gpurun_out/r02/$T; mkdir -p $D
python scripts/stage_times.py --n 67108864 --reps 3 > $D/stages_c2.json 2>&1
python scripts/stage_times.py --n 16777216 --evrard --reps 3 > $D/stages_c3.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_build_warp|k_pass_item|k_pass_warp' -c 3 \
  -o $D/hot python scripts/stage_times.py --n 8388608 --reps 1 > $D/ncu_hot.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $D/launches_c2.csv python scripts/stage_times.py --n 67108864 --reps 1 > $D/ncu_launch.log 2>&1
echo done
