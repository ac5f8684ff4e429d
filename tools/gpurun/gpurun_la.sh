mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k lookahead 2>&1 | tail -3
for i in 1 2; do
for la in "" "--lookahead"; do
timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e $la > gpurun_out/bench_la$i$la.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/bench_la$i$la.json')); print('lookahead' if d['lookahead'] else 'serial   ', round(d['value'],3), 'TF', round(d['ms_per_step'],2), 'ms', d['clocks']['sm_mhz'])"
done; done
