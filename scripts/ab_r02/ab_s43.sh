#!/bin/bash
# LJ pass: two entries in flight (SFCNL_PW_TWO) at 4 / 3 CTAs per SM vs one
D=gpurun_out/r02/s43; mkdir -p $D
st() { SFCNL_LIB=abv/$1/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2; do st cur; st two4; st two3; done
echo done
