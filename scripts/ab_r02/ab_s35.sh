#!/bin/bash
# k_decode_store: index data staged in shared memory, next SC claimed one ahead (dec1) vs global byte loads (dec0)
D=gpurun_out/r02/s35; mkdir -p $D
st() { SFCNL_LIB=abv/$1/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2; do st dec0; st dec1; done
SFCNL_LIB=abv/dec1/libsfcnl_b200.so timeout 600 ncu --metrics gpu__time_duration.sum -k regex:k_decode_store --clock-control none --csv python scripts/stage_times.py --n 67108864 --reps 1 > $D/ncu_dec1.csv 2>&1
SFCNL_LIB=abv/dec1/libsfcnl_b200.so timeout 1500 python -m pytest tests/test_gpu_predecode.py tests/test_gpu_parity.py tests/test_gpu_errors.py tests/test_gpu_edge.py tests/test_gpu_x64.py -x -q -p no:cacheprovider > $D/parity.txt 2>&1
echo done
