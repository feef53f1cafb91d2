#!/bin/bash
# build: two-pass item rounds (first 1/2/3 rows of every item, then the rest of the open items)
D=gpurun_out/r02/s28; mkdir -p $D
st() { SFCNL_LIB=abv/$1/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2 3; do st head; st ph1; st ph2; st ph3; done
for v in ph1 ph2; do
SFCNL_LIB=abv/$v/libsfcnl_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fuzz.py -x -q -p no:cacheprovider > $D/parity_$v.txt 2>&1
done
echo done
