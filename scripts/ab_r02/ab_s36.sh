#!/bin/bash
# k_decode_store warp-strided (no per-SC atomic); k_halo_warp claiming 1 / 4 / 16 SCs per atomic
D=gpurun_out/r02/s36; mkdir -p $D
st() { SFCNL_LIB=abv/$1/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2; do st base; st hb1; st hb4; st hb16; done
for v in base hb1 hb4 hb16; do
SFCNL_LIB=abv/$v/libsfcnl_b200.so timeout 600 ncu --metrics gpu__time_duration.sum -k regex:'k_decode_store|k_halo_warp' --clock-control none --csv python scripts/stage_times.py --n 67108864 --reps 1 > $D/ncu_$v.csv 2>&1
done
SFCNL_LIB=abv/hb4/libsfcnl_b200.so timeout 1500 python -m pytest tests/test_gpu_predecode.py tests/test_gpu_parity.py tests/test_gpu_errors.py tests/test_gpu_edge.py tests/test_distributed.py -x -q -p no:cacheprovider > $D/parity.txt 2>&1
echo done
