#!/bin/bash
# density item pass: 4 / 5 / 6 CTAs per SM (128 / 96 / 80 registers)
D=gpurun_out/r02/s48; mkdir -p $D
st() { SFCNL_LIB=abv/$1/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2; do st c5; st c4; st c6; done
echo done
