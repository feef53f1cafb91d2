#!/bin/bash
# build: fp32 traversal pre-test (F 512 / 320); fp64 pass two slots per step
D=gpurun_out/r02/s6; mkdir -p $D
st() { SFCNL_LIB=abv/$1/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2; do st base; st tr512; st tr320; done
for v in base tr512 tr320; do SFCNL_BUILD_STATS=1 SFCNL_LIB=abv/$v/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 16777216 --evrard --reps 2 --label ${v}_c3 >> $D/ab.jsonl 2>> $D/ab.err; done
timeout 600 python scripts/stage_times.py --n 16777216 --reps 2 --f64 --label x64two_16 >> $D/ab.jsonl 2>>$D/ab.err
timeout 1500 python -m pytest tests/test_gpu_x64.py tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fuzz.py tests/test_full_list.py tests/test_distributed.py tests/test_lj_coulomb.py tests/test_gpu_errors.py -x -q -p no:cacheprovider > $D/parity.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > $D/fullsize.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_pass_x64' -c 2 -o $D/x64 python scripts/stage_times.py --n 8388608 --reps 1 --f64 > $D/ncu.log 2>&1
echo done
