#!/bin/bash
# min_image wrap out of line; existing alternative layouts (LJ on the item kernel, density on the warp kernel)
D=gpurun_out/r02/s14; mkdir -p $D
st() { SFCNL_LIB=abv/$1/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $2 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2 3; do st base base; st mini mini; done
SFCNL_PASS_ITEM_LJ=1 st base lj_item
SFCNL_DENSITY_WARP=1 st base rho_warp
timeout 900 python -m pytest tests/test_gpu_x64.py -x -q -p no:cacheprovider > $D/x64.txt 2>&1
echo done
