#!/bin/bash
# compute-sanitizer memcheck / racecheck / initcheck / synccheck over the smoke step and
# the edge-case, error and fp64-pass suites (gather + symmetric, 8x8 / 8x4 / 1x1, mixed + fp64). Logs under
# gpurun_out/r02/sanitize/.
D=gpurun_out/r02/sanitize; mkdir -p $D
CS=/usr/local/cuda/bin/compute-sanitizer
SMOKE='import __graft_entry__ as g; g.smoke()'
for tool in memcheck racecheck initcheck synccheck; do
  timeout 900 $CS --tool $tool --error-exitcode 9 python -c "$SMOKE" > $D/smoke_$tool.log 2>&1
  echo "smoke $tool rc=$?" | tee -a $D/summary.txt
done
for tool in memcheck racecheck; do
  timeout 1500 $CS --tool $tool --error-exitcode 9 python -m pytest tests/test_gpu_edge.py tests/test_gpu_errors.py tests/test_gpu_x64.py tests/test_gpu_predecode.py -x -q -p no:cacheprovider \
    > $D/edge_$tool.log 2>&1
  echo "edge+errors+x64+predecode $tool rc=$? $(tail -1 $D/edge_$tool.log)" | tee -a $D/summary.txt
done
grep -h "ERROR SUMMARY" $D/*.log | sort | uniq -c | tee -a $D/summary.txt
