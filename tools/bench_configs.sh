#!/bin/bash
# All BASELINE.json configs on one B200 (run under gpurun from the repo root):
# our arm (device-timed value, e2e through the host API, live per-stage
# roofline, cpu_baseline) and the reference arm for each, one JSON line per run
# in gpurun_out/${TAG}_bench_C*.json and gpurun_out/${TAG}_ref_C*.json.
TAG=${1:-r02}
STEPS=${STEPS:-50}
run() {  # name, args...
  local name=$1; shift
  python bench.py --steps $STEPS --warmup 5 "$@" > gpurun_out/${TAG}_bench_${name}.log 2>&1
  tail -1 gpurun_out/${TAG}_bench_${name}.log > gpurun_out/${TAG}_bench_${name}.json
  if [ -z "$NO_REF" ]; then
    python bench.py --impl reference --steps 20 --warmup 3 "$@" > gpurun_out/${TAG}_ref_${name}.log 2>&1
    tail -1 gpurun_out/${TAG}_ref_${name}.log > gpurun_out/${TAG}_ref_${name}.json
  fi
}
run C1 --B 16 --batch 1
run C2 --B 64 --batch 64
run C3 --B 128 --batch 1
run C4 --B 256 --batch 1 --e2e-steps 3
run C5 --B 32 --batch 4096 --real --e2e-steps 2
echo configs done
