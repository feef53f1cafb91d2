#!/bin/bash
# passes: L2 prefetch of the next chunk's j records (SFCNL_PF_NEXT) vs none
D=gpurun_out/r02/s33; mkdir -p $D
st() { SFCNL_LIB=abv/$1/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2 3; do st pf0; st pf1; done
echo done
