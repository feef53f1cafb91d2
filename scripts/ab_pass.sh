#!/bin/bash
# A/B of a compile-time variant on one B200: bench stages with the current build, then
# with pass.cu rebuilt with EXTRA (e.g. -DSFCNL_PW_NOPREFETCH). ab_pass.sh OUT EXTRA [N]
D=gpurun_out/${1:-ab}
mkdir -p $D
N=${3:-67108864}
run() { timeout 600 python bench.py --steps 5 --warmup 3 --particles $N --no-cpu-baseline --e2e-steps 0 > $D/$1.txt 2>&1; python - $D/$1.txt $1 <<'PY'
import json,sys
for L in open(sys.argv[1]):
    if L.startswith('{'):
        d=json.loads(L); print(sys.argv[2], "ms/step", d["ms_per_step"], d["stages_ms"])
PY
}
run A
touch paper_2602_19873_b200/csrc/pass.cu paper_2602_19873_b200/csrc/build.cu
make -C paper_2602_19873_b200 EXTRA="$2" > $D/make.txt 2>&1 || tail -5 $D/make.txt
run B
