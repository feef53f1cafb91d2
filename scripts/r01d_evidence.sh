#!/bin/bash
# Round-1 (session 3, end) evidence: smoke, default bench line, reference arm.
D=gpurun_out/r01d
mkdir -p $D
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1; tail -2 $D/smoke.txt
timeout 900 python bench.py > $D/bench.txt 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $D/bench_ref.txt 2>&1
tail -1 $D/bench.txt | cut -c1-300
tail -1 $D/bench_ref.txt | cut -c1-200
