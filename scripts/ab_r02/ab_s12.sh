#!/bin/bash
# scalar d2 (FMUL/FFMA) in the build row test and the pass loads
D=gpurun_out/r02/s12; mkdir -p $D
st() { SFCNL_LIB=abv/$1/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2; do st base; st bws; st ljs2; st rhos2; st rhod2; done
echo done
