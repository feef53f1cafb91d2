#!/bin/bash
# onesweep tile: 8 / 10 / 12 / 14 keys per thread
D=gpurun_out/r02/s46; mkdir -p $D
st() { SFCNL_LIB=abv/$1/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2; do st s12; st s8; st s10; st s14; done
echo done
