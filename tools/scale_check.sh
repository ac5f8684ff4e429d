#!/bin/bash
# weak-scaling bench at N = 1, 2, ..., visible GPUs (torchrun for N > 1) + the NCCL tests
mkdir -p gpurun_out
NG=$(python -c "import torch; print(torch.cuda.device_count())")
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x 2>&1 | tail -3
for N in 1 2 4 8; do
  [ $N -gt $NG ] && break
  if [ $N -eq 1 ]; then
    timeout 900 python bench.py --no-cpu-baseline > gpurun_out/scale_n1.json 2> gpurun_out/scale_n1.err
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29500 + N)) bench.py --gpus $N --no-cpu-baseline > gpurun_out/scale_n$N.json 2> gpurun_out/scale_n$N.err
  fi
  python -c "
import json
d = json.load(open('gpurun_out/scale_n$N.json'))
print('N=%d value %.3f TF  ms/step %.2f  orth %.2e  res %.2e  e2e %.2f  clocks %s' % (d['n_gpus'], d['value'], d['ms_per_step'], d['orthogonality'], d['residual'], d['e2e']['value'], d['clocks']))
print('   allreduce ms/step %.3f' % d['kernel_breakdown']['allreduce']['ms_per_step'])
" || tail -3 gpurun_out/scale_n$N.err
done
