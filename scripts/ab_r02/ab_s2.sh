#!/bin/bash
# A/B of the bulk-copy build staging (session 2 of round 2)
D=gpurun_out/r02/s2; mkdir -p $D
for v in base bulk bulkf320 base bulkf320 bulk; do
  SFCNL_BUILD_STATS=1 SFCNL_LIB=abv/$v/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 3 --label $v >> $D/ab.jsonl 2>> $D/ab.err
done
for v in bulk bulkf320; do
  SFCNL_LIB=abv/$v/libsfcnl_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fuzz.py tests/test_full_list.py tests/test_distributed.py -x -q -p no:cacheprovider > $D/parity_$v.txt 2>&1
done
SFCNL_LIB=abv/bulkf320/libsfcnl_b200.so timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "store or cluster" > $D/fullsize_bulkf320.txt 2>&1
echo done
