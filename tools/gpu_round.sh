#!/bin/bash
# one GPU call: smoke, the whole -m gpu suite (full log), a default bench line
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout ${PYTEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q -rs -s --durations=25 ${PYTEST_ARGS} > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/gpu_tests.log | tail -15
if [ -z "$NO_BENCH" ]; then
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python - << 'PY'
import json
try:
    d = json.load(open("gpurun_out/bench.json"))
    print("value %.3f TF  ms/step %.2f  orth %.3e  res %.3e  e2e %s  frac %s" % (d["value"], d["ms_per_step"], d["orthogonality"], d["residual"], d.get("e2e", {}).get("value"), d.get("roofline", {}).get("frac")))
    for k, v in d["kernel_breakdown"].items():
        print(f"  {k:10s} {v['ms_per_step']:8.2f} ms  n={v['launches_per_step']:5.1f}  tf={v['tflops']}  gbs={v['hbm_gbs']}")
except Exception as e:
    print("no bench json", e)
PY
tail -3 gpurun_out/bench.err
fi
