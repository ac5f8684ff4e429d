mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_wide.py -q 2>&1 | tail -3
for c in ss1k ss12k; do
timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_d.json 2>/dev/null;
python -c "
import json; d=json.load(open('gpurun_out/bench_${c}_d.json')); print('$c G=1', round(d['value'],2), 'TF', round(d['ms_per_step'],2), 'ms', 'orth %.2e' % d['orthogonality'], {k: round(v['ms_per_step'],1) for k,v in d['kernel_breakdown'].items() if v['ms_per_step']>0})" 2>&1 | tail -1
done
