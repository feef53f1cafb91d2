set -x
D=gpurun_out/r02/s1; mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $D/gpu.txt
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $D/pytest_gpu.txt 2>&1
timeout 900 python bench.py > $D/bench.json 2> $D/bench.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > $D/bench_ref.json 2> $D/bench_ref.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_build_warp|k_pass_item|k_pass_warp' -c 3 \
  -o $D/hot python scripts/stage_times.py --n 8388608 --reps 1 > $D/ncu_hot.log 2>&1
echo done
