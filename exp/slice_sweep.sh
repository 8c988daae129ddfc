#!/bin/bash
# round-trip time with G in L2-sized shell slices (SGL_G_CHUNK_MB), B = 128 one function
for mb in 0 96 64 32; do
  echo "== SGL_G_CHUNK_MB=$mb"
  SGL_G_CHUNK_MB=$mb timeout 200 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 --e2e-callers 1 > gpurun_out/sl.log 2>&1
  tail -1 gpurun_out/sl.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), 'us', {k: round(v['ms']*1e3,1) for k,v in d['stages'].items()})"
done
