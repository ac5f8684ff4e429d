mkdir -p gpurun_out
for c in cfg4-256 cfg4-128 cfg5; do
for fm in 1048576 65536; do
if [ $c = cfg5 ] && [ $fm = 65536 ]; then continue; fi
TSQR_FUSE_MAX=$fm timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29824 bench.py --gpus 4 --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_g4_fm$fm.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/bench_${c}_g4_fm$fm.json')); print('$c G=4 fuse_max=$fm', round(d['value'],2), 'TF', round(d['ms_per_step'],2), 'ms', 'orth %.2e' % d['orthogonality'], {k: round(v['ms_per_step'],1) for k,v in d['kernel_breakdown'].items() if v['ms_per_step']>0}, d['clocks']['sm_mhz'])" 2>&1 | tail -1
done; done
