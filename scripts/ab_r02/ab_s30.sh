#!/bin/bash
# keygen: exact shortcuts around the fp64 divisions (wrap skip, reciprocal cell with a guarded fallback)
D=gpurun_out/r02/s30; mkdir -p $D
st() { SFCNL_LIB=abv/$1/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2 3; do st head; st keyfast; done
SFCNL_LIB=abv/keyfast/libsfcnl_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_edge.py -x -q -p no:cacheprovider > $D/parity.txt 2>&1
SFCNL_LIB=abv/keyfast/libsfcnl_b200.so timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "sfc_order" > $D/fullsize.txt 2>&1
echo done
