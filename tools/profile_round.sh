#!/bin/bash
# Round profile on one B200 (run under gpurun from the repo root):
#   1. every BASELINE config's bench line and reference-arm line (tools/bench_configs.sh),
#   2. the ncu launch list of a short bench run of every config,
#   3. one ncu --set full capture of a B = 128 round trip (all six kernels).
# Outputs land in gpurun_out/; tools/profile_summaries.py writes profiles/ from them.
R=${1:-r02}
bash tools/bench_configs.sh $R
for cfg in "C1 --B 16 --batch 1" "C2 --B 64 --batch 64" "C3 --B 128 --batch 1" "C4 --B 256 --batch 1" "C5 --B 32 --batch 4096 --real"; do
  set -- $cfg; name=$1; shift
  ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
      --log-file gpurun_out/${R}_launches_${name}.csv python bench.py "$@" --steps 2 --warmup 3 --no-cpu-baseline \
      --e2e-steps 1 --e2e-callers 1 > gpurun_out/${R}_ncu_launch_${name}.log 2>&1
done
cp gpurun_out/${R}_launches_C3.csv gpurun_out/${R}_launches.csv
ncu --set full --import-source on --clock-control none -k regex:"az_|gemm_dmma|leginv_wp|radfwd_wp" -c 6 \
    -o gpurun_out/${R}_full -f python tools/profile_step.py --steps 1 > gpurun_out/${R}_ncu_full.log 2>&1
echo profile done
