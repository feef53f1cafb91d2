#!/bin/bash
# LJ entry loop: pinned j-quarter shared base (1 IMAD per entry instead of 3) and the
# shorter energy / force chain (s6 - 1 reused) vs the previous form (SFCNL_PW_OLD).
D=gpurun_out/ab_lj_v3; mkdir -p $D
for v in base v3 base v3 base v3; do
  SFCNL_LIB=abv/$v/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 3 --label $v >> $D/stages.jsonl 2>> $D/err.txt
done
SFCNL_LIB=abv/v3/libsfcnl_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_lj_coulomb.py tests/test_gpu_edge.py tests/test_gpu_fuzz.py tests/test_gpu_predecode.py -x -q > $D/pytest_v3.txt 2>&1; tail -2 $D/pytest_v3.txt
SFCNL_LIB=abv/v3/libsfcnl_b200.so timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "lj" > $D/pytest_full_v3.txt 2>&1; tail -2 $D/pytest_full_v3.txt
