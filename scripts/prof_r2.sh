#!/bin/bash
# ncu --set full of the build + pass kernels on an 8M step
D=gpurun_out/${1:-prof}
mkdir -p $D
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${3:-k_build_smem|k_pass_warp}" -c 3 -o $D/full python scripts/prof_pass.py ${2:-8388608} > $D/ncu_full.log 2>&1
tail -3 $D/ncu_full.log
