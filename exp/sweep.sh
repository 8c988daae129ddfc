#!/bin/bash
# usage: exp/sweep.sh tag "ENV=.. ENV2=.." ["ENV=.."] ...  (runs on the GPU box)
tag=$1; shift
for cfg in "$@"; do
  env $cfg python bench.py --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 1 "${BENCH_ARGS[@]}" $BARGS > gpurun_out/sw.log 2>&1
  python - "$cfg" <<'PY' >> gpurun_out/${tag}_sweep.txt
import json,sys
l=[x for x in open('gpurun_out/sw.log') if x.startswith('{')]
if not l: print(sys.argv[1], 'FAILED', open('gpurun_out/sw.log').read()[-500:]); sys.exit()
d=json.loads(l[-1]); st=d.get('stages',{})
print(f"{sys.argv[1]:40s} {d['ms_per_step']*1e3:8.1f} us  "+" ".join(f"{k[:6]}={v['ms']*1e3:.1f}" for k,v in st.items()))
PY
done
cat gpurun_out/${tag}_sweep.txt
