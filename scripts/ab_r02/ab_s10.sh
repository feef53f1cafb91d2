#!/bin/bash
# onesweep ranking: match_any vs per-bit ballots; 2 vs 3 CTAs per SM
D=gpurun_out/r02/s10; mkdir -p $D
st() { SFCNL_LIB=abv/$1/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2; do st base; st sortb; st sortb3; st sort3; done
for v in sortb3 sort3; do
SFCNL_LIB=abv/$v/libsfcnl_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -p no:cacheprovider -k "sort or pipeline or fuzz" > $D/parity_$v.txt 2>&1
done
for r in 1 2; do for v in px2 px3 px4; do SFCNL_LIB=abv/$v/libsfcnl_b200.so timeout 600 python scripts/stage_times.py --n 16777216 --reps 2 --f64 --label $v >> $D/ab.jsonl 2>>$D/ab.err; done; done
SFCNL_LIB=abv/px4/libsfcnl_b200.so timeout 900 python -m pytest tests/test_gpu_x64.py -x -q -p no:cacheprovider > $D/x64_px4.txt 2>&1
SFCNL_LIB=abv/px3/libsfcnl_b200.so timeout 900 python -m pytest tests/test_gpu_x64.py -x -q -p no:cacheprovider > $D/x64_px3.txt 2>&1
echo done2
