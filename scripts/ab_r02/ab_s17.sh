#!/bin/bash
# build: near-first item order (homogeneous rounds for the early-exit row loop); exact node test out of line
D=gpurun_out/r02/s17; mkdir -p $D
st() { SFCNL_LIB=abv/$1/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2 3; do st head; st near; st nodeol; done
for v in head near; do SFCNL_LIB=abv/$v/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 16777216 --evrard --reps 2 --label ${v}_c3 >> $D/ab.jsonl 2>> $D/ab.err; done
SFCNL_LIB=abv/near/libsfcnl_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fuzz.py -x -q -p no:cacheprovider > $D/parity_near.txt 2>&1
echo done
