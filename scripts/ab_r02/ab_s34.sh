#!/bin/bash
# passes: pass-to-pass row culling (density records row bits, LJ skips rows) vs off
D=gpurun_out/r02/s34; mkdir -p $D
st() { timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2 3; do SFCNL_NO_ROWCULL=1 st off; st rowcull; done
timeout 1500 python -m pytest tests/test_gpu_predecode.py tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_errors.py tests/test_lj_coulomb.py tests/test_gpu_fuzz.py -x -q -p no:cacheprovider > $D/parity.txt 2>&1
echo done
