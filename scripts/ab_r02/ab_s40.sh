#!/bin/bash
# apply_sfc_order: shared-memory staged record pack + 16-byte record gather (perm1) vs per-double (perm0)
D=gpurun_out/r02/s40; mkdir -p $D
st() { SFCNL_LIB=abv/$1/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2 3; do st perm0; st perm1; done
for v in perm0 perm1; do
SFCNL_LIB=abv/$v/libsfcnl_b200.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:'_records' --clock-control none --csv python scripts/stage_times.py --n 67108864 --reps 1 > $D/ncu_$v.csv 2>&1
done
SFCNL_LIB=abv/perm1/libsfcnl_b200.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_edge.py tests/test_distributed.py tests/test_gpu_keygen.py -x -q -p no:cacheprovider > $D/parity.txt 2>&1
echo done
