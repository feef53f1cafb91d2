#!/bin/bash
# onesweep tile: 12 / 16 / 20 / 24 keys per thread
D=gpurun_out/r02/s45; mkdir -p $D
st() { SFCNL_LIB=abv/$1/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2; do st s16; st s12; st s20; st s24; done
echo done
