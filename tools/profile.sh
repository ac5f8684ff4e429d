#!/bin/bash
# ncu evidence: launch list of our kernels (-k regex:^k_) and full captures of selected kernels.
# usage: bash tools/profile.sh <tag> [kernel_regex:skip:count ...]
TAG=${1:-run}; shift
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/prof_${TAG}_plain.json 2> gpurun_out/prof_${TAG}_plain.err || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:^k_ --csv \
    --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launches_${TAG}.log 2>&1
for spec in "$@"; do
  IFS=: read -r K S C <<< "$spec"
  ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c $C \
      -o gpurun_out/prof_${TAG}_${K} $CMD > gpurun_out/ncu_${TAG}_${K}.log 2>&1
done
ls gpurun_out
