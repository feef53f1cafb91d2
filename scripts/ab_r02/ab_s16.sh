#!/bin/bash
# build: __builtin_expect on the unsafe / guard-band branches (block placement)
D=gpurun_out/r02/s16; mkdir -p $D
st() { SFCNL_LIB=abv/$1/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2 3; do st head; st expect; done
for v in head expect; do SFCNL_LIB=abv/$v/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 16777216 --evrard --reps 2 --label ${v}_c3 >> $D/ab.jsonl 2>> $D/ab.err; done
echo done
