#!/bin/bash
# ncu --set full of selected kernels on one uniform step: prof_r2.sh OUT N REGEX [SKIP] [COUNT]
D=gpurun_out/${1:-prof}
mkdir -p $D
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${3:-k_build_warp|k_pass}" -s ${4:-0} -c ${5:-3} -o $D/full python scripts/prof_pass.py ${2:-8388608} > $D/ncu_full.log 2>&1
tail -3 $D/ncu_full.log
