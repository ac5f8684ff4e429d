mkdir -p gpurun_out
N=$(python -c "import torch; print(torch.cuda.device_count())")
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_n$N.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_fused_plane.py -v -rs 2>&1 | tail -45 > gpurun_out/multi_tests_n$N.log; tail -8 gpurun_out/multi_tests_n$N.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
   bench.py --gpus $N --no-cpu-baseline > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo "bench rc=$?"
python - << PY
import json
d = json.load(open("gpurun_out/bench_n$N.json"))
print("N=%d value %.3f TF  ms/step %.2f  orth %.2e  res %.2e  e2e %s plane %s" % (d["n_gpus"], d["value"], d["ms_per_step"], d["orthogonality"], d["residual"], d["e2e"]["value"] if d.get("e2e") else None, d["config"]["data_plane"][:20]))
PY
