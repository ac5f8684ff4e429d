mkdir -p gpurun_out
for c in ss1k ss6k ss12k; do
for G in 1 2 4; do
if [ $G = 1 ]; then CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_g$G.json 2> gpurun_out/bench_${c}_g$G.err;
else CUDA_VISIBLE_DEVICES=$(python -c "print(','.join(str(i) for i in range($G)))") timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port 2961$G bench.py --gpus $G --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_g$G.json 2> gpurun_out/bench_${c}_g$G.err; fi
python -c "
import json; d=json.load(open('gpurun_out/bench_${c}_g$G.json')); print('$c G=$G', round(d['value'],2), 'TF', round(d['ms_per_step'],2), 'ms', 'orth %.2e res %.2e' % (d['orthogonality'], d['residual']), {k: round(v['ms_per_step'],1) for k,v in d['kernel_breakdown'].items() if v['ms_per_step']>0}, d['clocks']['sm_mhz'])" 2>&1 | tail -1
done; done
