#!/bin/bash
# density item pass: saturated scalar fmas for max(1 - q, 0), max(1/2 - q, 0) vs the
# packed form + FMNMX (SFCNL_PI_OLD)
D=gpurun_out/ab_density_sat; mkdir -p $D
for v in base sat base sat base sat; do
  SFCNL_LIB=abv/$v/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 3 --label $v >> $D/stages.jsonl 2>> $D/err.txt
done
SFCNL_LIB=abv/sat/libsfcnl_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fuzz.py tests/test_gpu_predecode.py tests/test_gpu_scale.py -x -q > $D/pytest_sat.txt 2>&1; tail -2 $D/pytest_sat.txt
SFCNL_LIB=abv/sat/libsfcnl_b200.so timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "density" > $D/pytest_full_sat.txt 2>&1; tail -2 $D/pytest_full_sat.txt
