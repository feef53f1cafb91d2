#!/bin/bash
# apply_sfc_order: 48-byte records (perm1) vs 64-byte padded records (pad); world-1 NCCL DD test
D=gpurun_out/r02/s41; mkdir -p $D
st() { SFCNL_LIB=abv/$1/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2; do st perm1; st pad; done
for v in perm1 pad; do
SFCNL_LIB=abv/$v/libsfcnl_b200.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:'_records' --clock-control none --csv python scripts/stage_times.py --n 67108864 --reps 1 > $D/ncu_$v.csv 2>&1
done
timeout 1500 python -m pytest tests/test_distributed.py -x -q -p no:cacheprovider > $D/dist.txt 2>&1
echo done
