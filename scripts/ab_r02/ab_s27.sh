#!/bin/bash
# build: near-first item rounds on the cached-leaf tier
D=gpurun_out/r02/s27; mkdir -p $D
st() { SFCNL_LIB=abv/$1/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2 3; do st head; st near; done
SFCNL_LIB=abv/near/libsfcnl_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fuzz.py -x -q -p no:cacheprovider > $D/parity.txt 2>&1
echo done
