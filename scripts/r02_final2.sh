#!/bin/bash
# End-of-round evidence (session 3) on one B200: full GPU suite, smoke, bench (b200 arm; the
# reference arm is unchanged), ncu launch list of a C2 step, one --set full capture at C2.
D=gpurun_out/r02/final2; mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $D/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $D/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1
timeout 900 python bench.py > $D/bench.json 2> $D/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $D/launches_c2.csv python scripts/stage_times.py --n 67108864 --reps 1 > $D/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_pass_warp|k_build_warp|k_pass_item' -c 3 \
  -o $D/hot_c2 python scripts/stage_times.py --n 67108864 --reps 1 > $D/ncu_hot.log 2>&1
echo done
