#!/bin/bash
# Round profile on one B200 (run under gpurun from the repo root):
#   1. the bench line (no profiler), 2. the ncu launch list of a short bench run,
#   3. one ncu --set full capture of a B = 128 round trip (all six kernels).
# Outputs land in gpurun_out/; the summaries are copied into profiles/ by hand.
set -e
R=${1:-r01}
python bench.py > gpurun_out/${R}_bench.log 2>&1
tail -1 gpurun_out/${R}_bench.log > gpurun_out/${R}_bench.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${R}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
    > gpurun_out/${R}_ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"az_|gemm_dmma" -c 6 \
    -o gpurun_out/${R}_full -f python tools/profile_step.py --steps 1 > gpurun_out/${R}_ncu_full.log 2>&1
echo profile done
