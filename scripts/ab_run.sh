for v in base v1 v1two base v1; do SFCNL_LIB=abv/$v/libsfcnl_b200.so python scripts/stage_times.py --n 67108864 --reps 3 --label $v; done
SFCNL_LIB=abv/v1/libsfcnl_b200.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_lj_coulomb.py -x -q 2>&1 | tail -3
