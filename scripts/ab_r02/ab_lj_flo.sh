#!/bin/bash
# LJ entry loop control: highest entry first (FLO + BMSK) vs lowest first (BREV + FLO,
# SFCNL_PW_FFS); both builds carry the saturated-fma density spline
D=gpurun_out/ab_lj_flo; mkdir -p $D
for v in ffs flo ffs flo ffs flo; do
  SFCNL_LIB=abv/$v/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 3 --label $v >> $D/stages.jsonl 2>> $D/err.txt
done
SFCNL_LIB=abv/flo/libsfcnl_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_lj_coulomb.py tests/test_gpu_edge.py tests/test_gpu_fuzz.py tests/test_gpu_predecode.py tests/test_full_list.py -x -q > $D/pytest_flo.txt 2>&1; tail -2 $D/pytest_flo.txt
SFCNL_LIB=abv/flo/libsfcnl_b200.so timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "mixed" > $D/pytest_full_flo.txt 2>&1; tail -2 $D/pytest_full_flo.txt
