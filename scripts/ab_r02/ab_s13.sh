#!/bin/bash
# density pass: per-chunk fp32 running sums instead of a per-round fp64 update
D=gpurun_out/r02/s13; mkdir -p $D
st() { SFCNL_LIB=abv/$1/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2 3; do st base; st runsum; done
SFCNL_LIB=abv/runsum/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 16777216 --evrard --reps 2 --label runsum_c3 >> $D/ab.jsonl 2>> $D/ab.err
SFCNL_LIB=abv/base/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 16777216 --evrard --reps 2 --label base_c3 >> $D/ab.jsonl 2>> $D/ab.err
SFCNL_LIB=abv/runsum/libsfcnl_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fuzz.py tests/test_full_list.py -x -q -p no:cacheprovider > $D/parity.txt 2>&1
SFCNL_LIB=abv/runsum/libsfcnl_b200.so timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k mixed > $D/fullsize.txt 2>&1
echo done
