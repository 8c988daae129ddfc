#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for b in 128 64 256; do timeout 300 tools/e2e_dropin $b 6 2; done
python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 10 > gpurun_out/e2e_c3.log 2>&1; tail -1 gpurun_out/e2e_c3.log | cut -c1-200
python - <<'PY'
import json
d=json.loads(open('gpurun_out/e2e_c3.log').read().strip().splitlines()[-1])
print('C3 value', d['value'], 'e2e', d['e2e'])
PY
python bench.py --B 64 --batch 64 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 4 > gpurun_out/e2e_c2.log 2>&1
python - <<'PY'
import json
d=json.loads(open('gpurun_out/e2e_c2.log').read().strip().splitlines()[-1])
print('C2 value', d['value'], 'e2e', d['e2e'])
PY
