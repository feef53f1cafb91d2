#!/bin/bash
# LJ pass: close pairs (< 1.22 sigma) out of line into fp64 side sums; with 4 / 5 CTAs per SM
D=gpurun_out/r02/s29; mkdir -p $D
st() { SFCNL_LIB=abv/$1/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2 3; do st head; st ljclose; st ljclose5; done
SFCNL_LIB=abv/ljclose/libsfcnl_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_lj_coulomb.py -x -q -p no:cacheprovider > $D/parity.txt 2>&1
echo done
