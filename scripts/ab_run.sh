for v in base exp direct exp base; do SFCNL_LIB=abv/$v/libsfcnl_b200.so python scripts/stage_times.py --n 67108864 --reps 3 --label $v; done
SFCNL_LIB=abv/exp/libsfcnl_b200.so python scripts/stage_times.py --n 16777216 --evrard --reps 2 --label exp_c3
SFCNL_LIB=abv/exp/libsfcnl_b200.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fuzz.py tests/test_full_list.py tests/test_store_file.py -x -q 2>&1 | tail -2
SFCNL_LIB=abv/exp/libsfcnl_b200.so python -m pytest tests/test_gpu_fullsize.py -x -q -k "C3 and (store or cluster)" 2>&1 | tail -2
