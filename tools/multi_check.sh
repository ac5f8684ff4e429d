#!/bin/bash
# multi-GPU checks: NCCL tests + weak-scaling bench at N = number of visible GPUs
mkdir -p gpurun_out
N=$(python -c "import torch; print(torch.cuda.device_count())")
echo "gpus=$N"
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x 2>&1 | tail -8 > gpurun_out/multi_tests.log; cat gpurun_out/multi_tests.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
   bench.py --gpus $N --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo "bench rc=$?"
python - << PY
import json
try:
    d = json.load(open("gpurun_out/bench_n$N.json"))
    print("N=%d value %.3f TF  ms/step %.2f  orth %.2e  res %.2e  e2e %s" % (d["n_gpus"], d["value"], d["ms_per_step"], d["orthogonality"], d["residual"], d["e2e"]["value"] if d.get("e2e") else None))
    for k, v in d["kernel_breakdown"].items():
        print(f"  {k:10s} {v['ms_per_step']:8.2f} ms  n={v['launches_per_step']:5.1f}")
except Exception as e:
    print("no bench json", e)
PY
tail -5 gpurun_out/bench_n$N.err
