mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_adaptive.py tests/test_gpu_cluster.py -q -x 2>&1 | tail -15 > gpurun_out/adapt_tests.log; tail -15 gpurun_out/adapt_tests.log
for a in mcqr2gs_adaptive; do
timeout 300 python - <<'PY' 2>&1 | tail -5
import sys, torch; sys.path.insert(0,'.')
import paper_2405_04237_b200 as t, synth
m,n,b=1<<22,512,64
for kappa in (1e2, 1e4, 1e15):
    A=t.colmajor_empty(m,n); synth.generate_torch(A,m,0,n,kappa,seed=0); A0=A.clone()
    for algo in ("mcqr2gs","mcqr2gs_adaptive"):
        p=t.Plan(m,n,b,algo); 
        for _ in range(2): A.copy_(A0); p.factor(A)
        e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        A.copy_(A0); torch.cuda.synchronize(); e0.record(); p.factor(A, wait=False); e1.record(); p.wait(); torch.cuda.synchronize()
        print(f"kappa={kappa:.0e} {algo:18s} {e0.elapsed_time(e1):8.2f} ms skipped={p.skipped_panels() if algo.endswith('adaptive') else 0}")
        p.close()
PY
done
