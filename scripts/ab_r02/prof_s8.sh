#!/bin/bash
# ncu --set full of the streaming kernels (keygen, one onesweep pass, permute) at C2
D=gpurun_out/r02/s8; mkdir -p $D
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_keygen|k_onesweep|k_gather_records|k_pack_records' -c 5 \
  -o $D/stream python scripts/stage_times.py --n 67108864 --reps 1 > $D/ncu.log 2>&1
echo done
