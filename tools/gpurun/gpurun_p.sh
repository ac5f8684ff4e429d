mkdir -p gpurun_out
export PATH=$PATH:/usr/local/cuda/bin
CONFIG=cfg3 bash tools/profile.sh r02_cfg3 launches > /dev/null 2>&1; echo "cfg3 launches rc=$?"
CONFIG=cfg3 bash tools/profile.sh r02_cfg3 full 'k_update_pp|k_proj' 4 > /dev/null 2>&1; echo "cfg3 full rc=$?"
python tools/profile_summary.py r02_cfg3 cfg3 > gpurun_out/summary_r02_cfg3.txt 2>&1
CONFIG=cfg1 bash tools/profile.sh r02_cfg1 launches > /dev/null 2>&1; echo "cfg1 launches rc=$?"
CONFIG=cfg1 bash tools/profile.sh r02_cfg1 full 'k_cluster' 1 > /dev/null 2>&1; echo "cfg1 full rc=$?"
python tools/profile_summary.py r02_cfg1 cfg1 > gpurun_out/summary_r02_cfg1.txt 2>&1
CONFIG=cfg5 bash tools/profile.sh r02_cfg5 launches > /dev/null 2>&1; echo "cfg5 launches rc=$?"
python tools/profile_summary.py r02_cfg5 cfg5 > gpurun_out/summary_r02_cfg5.txt 2>&1
mkdir -p gpurun_out/prof_out && cp -r profiles/r02_cfg3 profiles/r02_cfg1 profiles/r02_cfg5 profiles/ncu_traffic_r01.json gpurun_out/prof_out/
ncu -i gpurun_out/prof_r02_cfg1_full.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_out/cluster_sass_source.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep gpurun_out/launches_*.csv
du -sh gpurun_out
