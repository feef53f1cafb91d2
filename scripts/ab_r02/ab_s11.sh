#!/bin/bash
# scalar (FMUL/FFMA) instead of packed (FMUL2/FFMA2) kernel chains: LJ and SPH density passes
D=gpurun_out/r02/s11; mkdir -p $D
st() { SFCNL_LIB=abv/$1/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2 3; do st base; st ljs; st rhos; done
for v in ljs rhos; do
SFCNL_LIB=abv/$v/libsfcnl_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_lj_coulomb.py -x -q -p no:cacheprovider > $D/parity_$v.txt 2>&1
done
echo done
