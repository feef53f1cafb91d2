#!/bin/bash
# density pass: no in-range mask on the kernel value at query scale >= 1 (nomask) vs masked
D=gpurun_out/r02/s44; mkdir -p $D
st() { SFCNL_LIB=abv/$1/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2 3; do st mask; st nomask; done
SFCNL_LIB=abv/nomask/libsfcnl_b200.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fuzz.py tests/test_gpu_fullsize.py -k "not C4_8x4 and not C4_1x1" -x -q -p no:cacheprovider > $D/parity.txt 2>&1
echo done
