#!/bin/bash
# Round-1 (session 3) evidence on one B200: default bench line, ncu launch list of one
# 2^26 step (time + DRAM bytes per launch), ncu --set full of the hot kernels (2^23 step).
D=gpurun_out/r01e
mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $D/gpu.txt
timeout 900 python bench.py > $D/bench.txt 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $D/bench_ref.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $D/launches.csv python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $D/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_build_warp|k_pass_item|k_pass_warp" -c 3 -o $D/full python scripts/prof_pass.py 8388608 > $D/ncu_full.log 2>&1
ls -la $D
tail -2 $D/bench.txt | cut -c1-600
