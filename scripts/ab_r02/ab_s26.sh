#!/bin/bash
# LJ pass at 5 CTAs/SM (96 registers, spills) vs 4 (128)
D=gpurun_out/r02/s26; mkdir -p $D
st() { SFCNL_LIB=abv/$1/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2 3; do st head; st lj5; done
echo done
