#!/bin/bash
# Round-1 evidence on one B200: full C2 bench line, ncu launch list of one 64M step,
# one ncu --set full capture of the build + pass kernels (8M step).
set -x
mkdir -p gpurun_out/r01
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r01/gpu.txt
timeout 900 python bench.py > gpurun_out/r01/bench.json 2> gpurun_out/r01/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r01/launches.csv python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r01/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_build_smem|k_pass_ws|k_onesweep|k_gather" -c 5 -o gpurun_out/r01/full python scripts/prof_pass.py 8388608 > gpurun_out/r01/ncu_full.log 2>&1
ls -la gpurun_out/r01
