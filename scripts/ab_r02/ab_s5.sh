#!/bin/bash
# build variants: expanded/difference pair test x cold paths out of line/inline, fp32 traversal pre-test
D=gpurun_out/r02/s5; mkdir -p $D
st() { SFCNL_LIB=abv/$1/libsfcnl_b200.so timeout 300 python scripts/stage_times.py --n 67108864 --reps 2 --label $2 >> $D/ab.jsonl 2>> $D/ab.err; }
for r in 1 2; do
  st base base; st exp_cold exp_cold; st exp_inl exp_inl; st diff_cold diff_cold; st diff_inl diff_inl
  SFCNL_TRAV_FP64=1 st exp_inl exp_inl_trav64
  SFCNL_TRAV_FP64=1 st diff_inl diff_inl_trav64
done
SFCNL_LIB=abv/exp_inl/libsfcnl_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fuzz.py tests/test_full_list.py tests/test_distributed.py -x -q -p no:cacheprovider > $D/parity_exp_inl.txt 2>&1
echo done
