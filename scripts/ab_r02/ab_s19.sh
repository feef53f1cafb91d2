#!/bin/bash
# LJ pass: fp32 per-i sums across chunks (fp64 only at the SC end)
D=gpurun_out/r02/s19; mkdir -p $D
st() { SFCNL_LIB=abv/$1/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2 3; do st head; st f32acc; done
SFCNL_LIB=abv/f32acc/libsfcnl_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_lj_coulomb.py -x -q -p no:cacheprovider > $D/parity.txt 2>&1
SFCNL_LIB=abv/f32acc/libsfcnl_b200.so timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "lj and (C2 or C3)" > $D/fullsize.txt 2>&1
echo done
