#!/bin/bash
# ncu evidence for one round, ONE ncu invocation per call (run the plain command first; ncu
# only if it exited 0):
#   [CONFIG=cfgN] bash tools/profile.sh <tag> launches -> launch list of our kernels (-k regex:^k_)
#   bash tools/profile.sh <tag> full <regex> <count> -> one --set full capture of <count>
#                                                     launches matching <regex>
# then `python tools/profile_summary.py <tag>` here.
TAG=${1:-run}; MODE=${2:-launches}
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --config ${CONFIG:-cfg3}"
$CMD > gpurun_out/prof_${TAG}_plain.json 2> gpurun_out/prof_${TAG}_plain.err || exit 1
if [ "$MODE" = launches ]; then
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:^k_ --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launches_${TAG}.log 2>&1
else
  K=$3; C=${4:-6}
  ncu --set full --clock-control none --import-source on -k regex:"$K" -c $C \
      -o gpurun_out/prof_${TAG}_full $CMD > gpurun_out/ncu_${TAG}_full.log 2>&1
fi
ls gpurun_out | grep "$TAG"
