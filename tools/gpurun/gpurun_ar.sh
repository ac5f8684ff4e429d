mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -q -k "factorisation and fused" 2>&1 | tail -2
for c in ss6k ss12k ss1k; do
for fm in 1048576 1000000000000; do
TSQR_FUSE_MAX=$fm timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29814 bench.py --gpus 4 --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_fm$fm.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/bench_${c}_fm$fm.json')); print('$c fuse_max=$fm', round(d['value'],2), 'TF', round(d['ms_per_step'],2), 'ms', {k: round(v['ms_per_step'],1) for k,v in d['kernel_breakdown'].items() if v['ms_per_step']>0})"
done; done
