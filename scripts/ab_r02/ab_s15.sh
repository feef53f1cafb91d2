#!/bin/bash
# min-image wrap out of line in the build / density / fp64 kernels, inline in the LJ pass's rare slots
D=gpurun_out/r02/s15; mkdir -p $D
st() { SFCNL_LIB=abv/$1/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2 3; do st base; st mini2; done
for v in base mini2; do SFCNL_LIB=abv/$v/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 16777216 --evrard --reps 2 --label ${v}_c3 >> $D/ab.jsonl 2>> $D/ab.err; done
SFCNL_LIB=abv/mini2/libsfcnl_b200.so timeout 600 python scripts/stage_times.py --n 16777216 --reps 2 --f64 --label mini2_f64 >> $D/ab.jsonl 2>> $D/ab.err
SFCNL_LIB=abv/mini2/libsfcnl_b200.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fuzz.py tests/test_full_list.py tests/test_distributed.py tests/test_gpu_x64.py tests/test_lj_coulomb.py tests/test_gpu_errors.py -x -q -p no:cacheprovider > $D/parity.txt 2>&1
echo done
