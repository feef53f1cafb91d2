#!/bin/bash
# passes: the store's index lists decoded once (k_decode_store) and shared by the density and LJ passes
D=gpurun_out/r02/s32; mkdir -p $D
st() { SFCNL_LIB=abv/cur/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2 3; do SFCNL_NO_PREDECODE=1 st inpass; st predecode; done
SFCNL_LIB=abv/cur/libsfcnl_b200.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_errors.py tests/test_gpu_fuzz.py tests/test_gpu_x64.py tests/test_distributed.py tests/test_lj_coulomb.py tests/test_store_file.py -x -q -p no:cacheprovider > $D/parity.txt 2>&1
echo done
