mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_cluster -c 1 -o gpurun_out/prof_cluster_cfg1b python bench.py --config cfg1 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_cluster.log 2>&1; echo "ncu rc=$?"
