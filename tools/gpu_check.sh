#!/bin/bash
# smoke + GPU tests + a short bench, each under its own timeout
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} 2>&1 | tail -15 > gpurun_out/gpu_tests.log; tail -6 gpurun_out/gpu_tests.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python - << 'PY'
import json
try:
    d = json.load(open("gpurun_out/bench.json"))
    print("value %.3f TF  ms/step %.2f  orth %.2e  res %.2e" % (d["value"], d["ms_per_step"], d["orthogonality"], d["residual"]))
    for k, v in d["kernel_breakdown"].items():
        print(f"  {k:10s} {v['ms_per_step']:8.2f} ms  n={v['launches_per_step']:5.1f}  tf={v['tflops']}  gbs={v['hbm_gbs']}")
except Exception as e:
    print("no bench json", e)
PY
tail -3 gpurun_out/bench.err
