#!/bin/bash
# build: fp32 traversal pre-test + 16-byte z rows + frontier 320 ("clean") vs base;
# LJ pass: software-pipelined entry loop (4 or 3 CTAs/SM)
D=gpurun_out/r02/s7; mkdir -p $D
st() { SFCNL_LIB=abv/$1/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2 3; do st base; st clean; st pipe; st pipe3; done
for v in base clean; do SFCNL_BUILD_STATS=1 SFCNL_LIB=abv/$v/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 16777216 --evrard --reps 2 --label ${v}_c3 >> $D/ab.jsonl 2>> $D/ab.err; done
SFCNL_LIB=abv/pipe/libsfcnl_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_lj_coulomb.py -x -q -p no:cacheprovider > $D/parity_pipe.txt 2>&1
echo done
