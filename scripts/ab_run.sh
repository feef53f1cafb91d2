python scripts/stage_times.py --n 16777216 --reps 2 --f64 --label x64_16m
SFCNL_EXACT_BLOCK=1 python scripts/stage_times.py --n 16777216 --reps 1 --f64 --label block_16m
python scripts/stage_times.py --n 67108864 --reps 2 --f64 --label x64_64m
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_edge.py tests/test_full_list.py -x -q 2>&1 | tail -3
python -m pytest tests/test_gpu_fullsize.py -x -q -k C3 2>&1 | tail -3
