#!/bin/bash
# build after the traversal kernel: main tier with / without traversal code, 5 / 6 CTAs
D=gpurun_out/r02/s24; mkdir -p $D
st() { SFCNL_LIB=abv/$1/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2 3; do st cur; st nobfs; st nobfs6; done
for v in cur nobfs nobfs6; do SFCNL_BUILD_STATS=1 SFCNL_LIB=abv/$v/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 16777216 --evrard --reps 2 --label ${v}_c3 >> $D/ab.jsonl 2>> $D/ab.err; done
for v in nobfs nobfs6; do
SFCNL_LIB=abv/$v/libsfcnl_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fuzz.py tests/test_distributed.py -x -q -p no:cacheprovider > $D/parity_$v.txt 2>&1
done
echo done
