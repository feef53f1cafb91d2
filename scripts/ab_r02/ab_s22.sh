#!/bin/bash
# build: traversal as a separate kernel (leaf cache) before the mask/encode kernel
D=gpurun_out/r02/s22; mkdir -p $D
st() { SFCNL_LIB=abv/cur/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $1 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2 3; do st head; SFCNL_PRETRAVERSE=1 st pretrav; done
SFCNL_PRETRAVERSE=1 SFCNL_LIB=abv/cur/libsfcnl_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fuzz.py -x -q -p no:cacheprovider > $D/parity.txt 2>&1
SFCNL_PRETRAVERSE=1 SFCNL_LIB=abv/cur/libsfcnl_b200.so timeout 600 ncu --set full --clock-control none -k regex:'k_build_warp|k_halo_warp' -c 2 -o $D/pretrav python scripts/stage_times.py --n 8388608 --reps 1 > $D/ncu.log 2>&1
echo done
