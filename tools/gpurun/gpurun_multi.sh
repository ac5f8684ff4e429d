mkdir -p gpurun_out
N=$(python -c "import torch; print(torch.cuda.device_count())")
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_n$N.txt 2>&1
timeout 1800 python -m pytest tests/test_gpu_multi.py -v -rs 2>&1 | tail -30 > gpurun_out/multi_tests_n$N.log; tail -4 gpurun_out/multi_tests_n$N.log
for G in 1 2 $N; do
if [ $G = 1 ]; then CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_g$G.json 2> gpurun_out/bench_g$G.err;
else
CUDA_VISIBLE_DEVICES=$(python -c "print(','.join(str(i) for i in range($G)))") timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port 2951$G \
   bench.py --gpus $G --no-cpu-baseline > gpurun_out/bench_g$G.json 2> gpurun_out/bench_g$G.err; fi
echo "bench G=$G rc=$?"
python - << PY
import json
d = json.load(open("gpurun_out/bench_g$G.json"))
print("N=%d value %.3f TF  ms/step %.2f  orth %.2e  res %.2e  e2e %s plane %s clocks %s" % (d["n_gpus"], d["value"], d["ms_per_step"], d["orthogonality"], d["residual"], d["e2e"]["value"] if d.get("e2e") else None, d["config"]["data_plane"][:20], d.get("clocks")))
PY
done
