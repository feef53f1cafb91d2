#!/bin/bash
# build: expanded-form pair test + smaller main-tier frontier; LJ predicate trim
D=gpurun_out/r02/s4; mkdir -p $D
for v in base new base new; do
  SFCNL_BUILD_STATS=1 SFCNL_LIB=abv/$v/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 3 --label $v >> $D/ab.jsonl 2>> $D/ab.err
done
for v in base new; do
  SFCNL_BUILD_STATS=1 SFCNL_LIB=abv/$v/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 16777216 --evrard --reps 3 --label ${v}_c3 >> $D/ab.jsonl 2>> $D/ab.err
done
SFCNL_LIB=abv/new/libsfcnl_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fuzz.py tests/test_full_list.py tests/test_distributed.py tests/test_gpu_x64.py -x -q -p no:cacheprovider > $D/parity_new.txt 2>&1
SFCNL_LIB=abv/new/libsfcnl_b200.so timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > $D/fullsize_new.txt 2>&1
SFCNL_LIB=abv/new/libsfcnl_b200.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_build_warp' -c 1 -o $D/build python scripts/stage_times.py --n 8388608 --reps 1 > $D/ncu.log 2>&1

SFCNL_LIB=abv/new/libsfcnl_b200.so timeout 600 python scripts/stage_times.py --n 16777216 --reps 3 --f64 --label new16_f64 >> $D/ab.jsonl 2>>$D/ab.err
SFCNL_LIB=abv/new/libsfcnl_b200.so timeout 600 python scripts/stage_times.py --n 67108864 --reps 2 --f64 --label new64_f64 >> $D/ab.jsonl 2>>$D/ab.err
echo done
