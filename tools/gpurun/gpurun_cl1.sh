mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cluster.py -q 2>&1 | tail -2
for i in 1 2; do
timeout 300 python bench.py --config cfg1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
python -c "
import json; d=json.load(open('gpurun_out/bench_cfg1.json')); print(d['exec_path'], d['ms_per_step'], d['value'], d['orthogonality'], d['e2e']['ms_per_step'])"
done
