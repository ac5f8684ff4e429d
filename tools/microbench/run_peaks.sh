#!/bin/bash
# Runs the FP64 peak microbenchmarks on a B200 and records clocks during the run.
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.sw_power_cap --format=csv -lms 200 -i 0 > gpurun_out/peaks_clocks.csv &
SMI=$!
./tools/microbench/fp64_peaks > gpurun_out/fp64_peaks.json 2> gpurun_out/fp64_peaks.err
python - >> gpurun_out/fp64_peaks_torch.json << 'PY'
import torch, time, json
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
for _ in range(3): a @ b
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(10):
    e0.record(); a @ b; e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
t0 = time.time(); n = 0
e0.record()
while time.time() - t0 < 4:
    a @ b; n += 1
e1.record(); torch.cuda.synchronize()
print(json.dumps({"dgemm_8192_burst_tflops": 2*8192**3/best/1e9, "dgemm_8192_sustained_tflops": 2*8192**3*n/e0.elapsed_time(e1)/1e9}))
PY
kill $SMI
nvidia-smi -q | grep -i -A3 "Clocks Event" > gpurun_out/peaks_smi.txt; nvidia-smi >> gpurun_out/peaks_smi.txt
lscpu | head -20 > gpurun_out/host_cpu.txt; nproc >> gpurun_out/host_cpu.txt; free -g >> gpurun_out/host_cpu.txt
