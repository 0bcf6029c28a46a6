#!/bin/bash
# Round profile (run under gpurun): plain bench, ncu launch list of the same
# command, one full ncu capture of the dominant kernel (run_kernel).
set -e
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2"
$CMD > gpurun_out/bench_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/launches_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:run_kernel -s 3 -c 1 \
    -o gpurun_out/prof_run -f $CMD > gpurun_out/ncu_full.log 2>&1
echo profile done
