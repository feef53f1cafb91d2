#!/bin/bash
# traversal kernel: 3 vs 6 CTAs/SM; ncu of the split build at 2^23
D=gpurun_out/r02/s25; mkdir -p $D
st() { SFCNL_LIB=abv/$1/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2 3; do st head; st nobfs_t6; done
SFCNL_LIB=abv/head/libsfcnl_b200.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_build_warp|k_halo_warp' -c 2 -o $D/split python scripts/stage_times.py --n 8388608 --reps 1 > $D/ncu.log 2>&1
echo done
