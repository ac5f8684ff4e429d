mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_wide.py -q -s 2>&1 | tail -6 > gpurun_out/wide_tests.log; tail -6 gpurun_out/wide_tests.log
for c in ss12k ss1k; do
timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_g1.json 2> gpurun_out/bench_${c}_g1.err;
python -c "
import json; d=json.load(open('gpurun_out/bench_${c}_g1.json')); print('$c G=1', d['scaling'], round(d['value'],2), 'TF', round(d['ms_per_step'],2), 'ms', 'orth %.2e res %.2e' % (d['orthogonality'], d['residual']), {k: round(v['ms_per_step'],1) for k,v in d['kernel_breakdown'].items() if v['ms_per_step']>0})" 2>&1 | tail -1
done
