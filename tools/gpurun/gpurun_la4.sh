mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -q -k lookahead 2>&1 | tail -3
for G in 4 2; do
for i in 1 2; do
for la in "" "--lookahead"; do
CUDA_VISIBLE_DEVICES=$(python -c "print(','.join(str(i) for i in range($G)))") timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port 2971$G bench.py --gpus $G --steps 6 --warmup 3 --no-cpu-baseline --no-e2e $la > gpurun_out/bench_la_g$G$i$la.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/bench_la_g$G$i$la.json')); print('G=$G', 'lookahead' if d['lookahead'] else 'serial   ', round(d['value'],3), 'TF', round(d['ms_per_step'],2), 'ms', d['clocks']['sm_mhz'], 'allreduce+chol ms', round(d['kernel_breakdown']['allreduce']['ms_per_step']+d['kernel_breakdown']['chol']['ms_per_step'],2))"
done; done; done
