#!/bin/bash
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_update -s 8 -c 1 \
    -o gpurun_out/prof2_update $CMD > gpurun_out/ncu2_update.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_proj -s 12 -c 1 \
    -o gpurun_out/prof2_proj $CMD > gpurun_out/ncu2_proj.log 2>&1
