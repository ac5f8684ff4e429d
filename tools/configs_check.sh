#!/bin/bash
mkdir -p gpurun_out
for c in cfg1 cfg2 cfg2-cqr2gs cfg5 cfg4-128 cfg4-256; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?"
  python -c "
import json
d=json.load(open('gpurun_out/bench_$c.json'))
print('  %s value %.3f TF ms/step %.3f orth %.2e res %.2e' % ('$c', d['value'], d['ms_per_step'], d['orthogonality'], d['residual']))
print('  ', {k: round(v['ms_per_step'],2) for k,v in d['kernel_breakdown'].items()})
" 2>&1 | tail -3
  tail -2 gpurun_out/bench_$c.err
done
