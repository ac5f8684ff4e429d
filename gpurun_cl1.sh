mkdir -p gpurun_out
./tools/microbench/chol_small
TSQR_LIB=paper_2405_04237_b200/libtsqr_prof.so timeout 300 python bench.py --config cfg1 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | grep CLPROF | tail -1
timeout 900 python -m pytest tests/test_gpu_cluster.py -q -x 2>&1 | tail -3
timeout 300 python bench.py --config cfg1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_cfg1.json')); print(d['exec_path'], d['ms_per_step'], d['value'], d['orthogonality'], d['residual'], d['e2e']['ms_per_step'])"
