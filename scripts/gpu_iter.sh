#!/bin/bash
# quick GPU iteration: parity tests + an 8M bench line (stage times)
D=gpurun_out/${1:-iter}
mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_distributed.py -x -q -m gpu > $D/pytest.txt 2>&1
tail -3 $D/pytest.txt
timeout 600 python bench.py --steps 3 --warmup 3 --particles ${2:-8388608} --no-cpu-baseline --e2e-steps 0 > $D/bench.txt 2>&1
python - $D/bench.txt <<'PY'
import json,sys
for L in open(sys.argv[1]):
    if L.startswith('{'):
        d=json.loads(L); print("ms/step", d["ms_per_step"], "ns/p", d["value"], d["stages_ms"])
PY
