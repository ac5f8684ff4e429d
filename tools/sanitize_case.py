"""Small factorisations for compute-sanitizer: cfg1 (4096 x 64, b = 16) and a
k = 3 case on the TMA paths (8192 + 64 rows x 192, b = 64), every algorithm once, plus the
blocked b = 128 Cholesky/TRMM path.  Usage:
    compute-sanitizer --tool memcheck python tools/sanitize_case.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2405_04237_b200 as t  # noqa: E402
import synth  # noqa: E402

cases = [(4096, 64, 16, 1e8, "mcqr2gs"), (8192 + 64, 192, 64, 1e12, "mcqr2gs"), (8192 + 64, 192, 64, 1e6, "cqr2gs"),
         (8192 + 64, 128, 128, 1e4, "cqr2"), (8192 + 64, 128, 128, 1e10, "scqr3"), (8192, 256, 128, 1e8, "mcqr2gs")]
for m, n, b, kappa, algo in cases:
    A, _, _ = synth.generate_np(m, n, kappa, seed=3, chunk=m)
    Ad = t.to_colmajor(A)
    R = t.factor(Ad, b, algo)
    torch.cuda.synchronize()
    print(f"{algo} {m}x{n} b={b}: R[0,0]={float(R[0, 0]):.6f}", flush=True)
print("sanitize cases done")
