#!/bin/bash
# fp64 pass (pass_x64.cuh) parity + timing; LJ predicate trim timing
D=gpurun_out/r02/s3; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_x64.py -x -q -p no:cacheprovider > $D/x64_tests.txt 2>&1
for r in 1 2; do
  timeout 600 python scripts/stage_times.py --n 16777216 --reps 3 --f64 --label new16 >> $D/st.jsonl 2>>$D/st.err
  SFCNL_PASS_EXACT_V1=1 timeout 600 python scripts/stage_times.py --n 16777216 --reps 2 --f64 --label v1_16 >> $D/st.jsonl 2>>$D/st.err
done
timeout 600 python scripts/stage_times.py --n 67108864 --reps 3 --f64 --label new64 >> $D/st.jsonl 2>>$D/st.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fuzz.py tests/test_lj_coulomb.py tests/test_gpu_errors.py -x -q -p no:cacheprovider > $D/parity.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "fp64 or lj" > $D/fullsize.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_pass_x64|k_pass_warp' -c 3 -o $D/x64 python scripts/stage_times.py --n 8388608 --reps 1 --f64 > $D/ncu.log 2>&1
echo done
