#!/bin/bash
# ncu evidence for round 1: launch list of our kernels (device time per launch) and a full
# capture of the top kernels. Plain run first (exit 0) as the profiling recipe requires.
set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tsqr --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_update -s 8 -c 2 \
    -o gpurun_out/prof_update $CMD > gpurun_out/ncu_update.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_atb -s 20 -c 3 \
    -o gpurun_out/prof_atb $CMD > gpurun_out/ncu_atb.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_trmm -s 6 -c 1 \
    -o gpurun_out/prof_trmm $CMD > gpurun_out/ncu_trmm.log 2>&1
ls -la gpurun_out
